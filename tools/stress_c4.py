"""Hang / determinism stress (development aid): mixed-size calls in one
context the way the test suite makes them, then repeated full C4 runs; every
C4 result must hash the same.  usage: python tools/stress_c4.py [reps]"""
import hashlib
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2002_04989_b200.engine import random_symmetric  # noqa: E402
from paper_2002_04989_b200 import IdentityEngine  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 6
eng = IdentityEngine()
a4 = random_symmetric(42, 4096) * np.sqrt(2.0 / 4096)
ref = None
for rep in range(reps):
    for n, lay in ((300, "narrow"), (1031, "wide8"), (1031, "widesp"), (300, "wide"), (2100, "")):
        if lay:
            os.environ["EIGENID_STAGE1_LAYOUT"] = lay
        else:
            os.environ.pop("EIGENID_STAGE1_LAYOUT", None)
        a = random_symmetric(5 + rep, n) * np.sqrt(2.0 / n)
        eng.minor_spectra(a, 0, min(n, 160))
    os.environ.pop("EIGENID_STAGE1_LAYOUT", None)
    t = time.time()
    g = eng.all_magnitudes(a4)
    h = hashlib.sha1(g.tobytes()).hexdigest()
    ref = ref or h
    print(f"rep {rep}: C4 {time.time() - t:.2f}s sha1={h[:16]} same={h == ref}", flush=True)
    assert h == ref
