"""SHA-1 of lambda(A) and minor spectra rows [0, R) of a seeded GOE matrix,
for checking that a kernel change is bit-identical (development aid).

usage: python tools/spectra_hash.py N R
"""
import hashlib
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2002_04989_b200.engine import random_symmetric  # noqa: E402
from paper_2002_04989_b200 import IdentityEngine  # noqa: E402

n, rows = int(sys.argv[1]), int(sys.argv[2])
a = random_symmetric(7, n) * np.sqrt(2.0 / n)
lam, mu = IdentityEngine().minor_spectra(a, 0, rows)
h = hashlib.sha1(np.ascontiguousarray(lam).tobytes() + np.ascontiguousarray(mu).tobytes())
print(f"n={n} rows={rows} sha1={h.hexdigest()}")
