"""Histogram of Sturm evaluations per eigenvalue in the minor bisection
(development aid; needs a build with -DEIGENID_BISECT_STATS, e.g.
VARIANT=-DEIGENID_BISECT_STATS bash tools/variant_run.sh tools/bisect_stats.py N R)."""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2002_04989_b200._native as nat  # noqa: E402
from paper_2002_04989_b200 import IdentityEngine  # noqa: E402
from paper_2002_04989_b200.engine import random_symmetric  # noqa: E402

n, rows = int(sys.argv[1]), int(sys.argv[2])
a = random_symmetric(42, n) * np.sqrt(2.0 / n)
eng = IdentityEngine()
lam, mu = eng.minor_spectra(a, 0, rows)
lib = nat.load()
h = (ctypes.c_ulonglong * 64)()
lib.eigenid_debug_bisect_hist(h)
h = np.array(h[:], dtype=np.float64)
tot = h.sum()
mean = (h * np.arange(64)).sum() / tot
print(f"eigenvalues {int(tot)}  mean secant/bisection steps {mean:.2f} (+2 bracket evaluations)")
print("  steps:count", {i: int(h[i]) for i in range(64) if h[i]})
