"""Profiling driver: lambda(A) + minor spectra rows [0, R) of a seeded GOE
matrix (stage 1 + stage 2 + bisection only).  usage: prof_minors.py N R"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2002_04989_b200.engine import random_symmetric  # noqa: E402
from paper_2002_04989_b200 import IdentityEngine  # noqa: E402

n, rows = int(sys.argv[1]), int(sys.argv[2])
a = random_symmetric(42, n) * np.sqrt(2.0 / n)
eng = IdentityEngine()
for rep in range(int(os.environ.get("PROF_REPS", "2"))):  # the first call is cold
    print(f"-- call {rep}", file=sys.stderr, flush=True)
    t = time.time()
    lam, mu = eng.minor_spectra(a, 0, rows)
print(f"n={n} rows={rows} wall={time.time() - t:.3f}s mu_sum={mu.sum():.6f}", flush=True)
