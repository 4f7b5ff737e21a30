"""Runs the all_magnitudes pipeline on a seeded GOE matrix (profiling driver).

usage: python tools/prof_pipeline.py N [REPS]
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2002_04989_b200.engine import random_symmetric  # noqa: E402
from paper_2002_04989_b200 import IdentityEngine  # noqa: E402

n = int(sys.argv[1])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
a = random_symmetric(42, n) * np.sqrt(2.0 / n)
eng = IdentityEngine()
for r in range(reps):
    t = time.time()
    out = eng.all_magnitudes(a)
    print(f"n={n} rep={r} wall={time.time() - t:.3f}s sum={out.sum():.6f}", flush=True)
