"""Eigenvalue accuracy of the device pipeline against LAPACK (numpy eigvalsh)
on sampled minors of a seeded GOE matrix (development aid).

usage: python tools/accuracy_check.py N ROWS [SAMPLES]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2002_04989_b200.engine import random_symmetric  # noqa: E402
from paper_2002_04989_b200 import IdentityEngine  # noqa: E402

n, rows = int(sys.argv[1]), int(sys.argv[2])
samples = int(sys.argv[3]) if len(sys.argv) > 3 else 3
a = random_symmetric(42, n) * np.sqrt(2.0 / n)
lam, mu = IdentityEngine().minor_spectra(a, 0, rows)
ref_lam = np.linalg.eigvalsh(a)
print(f"n={n} lambda(A): max |err| = {np.abs(lam - ref_lam).max():.3e}")
errs = []
for j in np.linspace(0, rows - 1, samples).astype(int):
    mj = np.delete(np.delete(a, j, 0), j, 1)
    e = np.abs(mu[j] - np.linalg.eigvalsh(mj)).max()
    errs.append(e)
    print(f"  minor {j}: max |err| = {e:.3e}", flush=True)
print(f"max over sampled minors: {max(errs):.3e}")
