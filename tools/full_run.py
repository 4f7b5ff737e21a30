"""One full all_magnitudes(n) through the public API with per-stage timing
(EIGENID_PROFILE=1) and the doubly-stochastic check (development aid).
usage: python tools/full_run.py N"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("EIGENID_PROFILE", "1")
from paper_2002_04989_b200.engine import random_symmetric  # noqa: E402
from paper_2002_04989_b200 import IdentityEngine  # noqa: E402

n = int(sys.argv[1])
a = random_symmetric(42, n) * np.sqrt(2.0 / n)
eng = IdentityEngine()
for rep in range(int(os.environ.get("FULL_REPS", "1"))):
    t = time.time()
    g = eng.all_magnitudes(a).reshape(n, n)
    print(f"n={n} rep={rep} wall={time.time() - t:.2f}s rowsum={np.max(np.abs(g.sum(1) - 1)):.2e} "
          f"colsum={np.max(np.abs(g.sum(0) - 1)):.2e}", flush=True)
