"""Profiling driver: identity kernel on C5-style spectra (n, rows)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2002_04989_b200 import IdentityEngine  # noqa: E402
from paper_2002_04989_b200.engine import c5_lambda  # noqa: E402

n, rows = int(sys.argv[1]), int(sys.argv[2])
eng = IdentityEngine()
lam = torch.from_numpy(c5_lambda(5, n)).cuda()
mu = torch.empty((rows, n - 1), dtype=torch.float64, device="cuda")
out = torch.empty((rows, n), dtype=torch.float64, device="cuda")
eng.c5_mu_device(5, lam.data_ptr(), n, 0, rows, mu.data_ptr())
for _ in range(2):
    eng.identity_device(lam.data_ptr(), mu.data_ptr(), n, 0, rows, out.data_ptr())
eng.sync()
print("ok", float(out.sum()))
