"""Small all_magnitudes runs for compute-sanitizer (one stage-1 layout per
run, chosen by EIGENID_STAGE1_LAYOUT): n = 200 exercises partial row blocks,
diagonal tiles, the panel_qr fallback and the helper launch.
usage: compute-sanitizer --tool racecheck python tools/sanitize_small.py [n]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2002_04989_b200.engine import random_symmetric  # noqa: E402
from paper_2002_04989_b200 import IdentityEngine  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
a = random_symmetric(3, n) * np.sqrt(2.0 / n)
g = IdentityEngine().all_magnitudes(a).reshape(n, n)
print(f"n={n} layout={os.environ.get('EIGENID_STAGE1_LAYOUT', 'default')} "
      f"rowsum={np.max(np.abs(g.sum(1) - 1)):.2e} colsum={np.max(np.abs(g.sum(0) - 1)):.2e}")
