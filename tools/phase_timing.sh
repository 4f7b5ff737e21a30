# Per-phase clock64 breakdown of stage 1 (CTA 0) and stage 2 (warp 0 of CTA 0)
# on a build with -DEIGENID_PHASE_TIMING (development aid, not the product).
set -e
cd $GRAFT_REPO_ROOT
mkdir -p /tmp/phb
for f in paper_2002_04989_b200/csrc/*.cu; do nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DEIGENID_PHASE_TIMING -Xcompiler -fPIC -c $f -o /tmp/phb/$(basename $f).o; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o /tmp/phb/libeigenid_b200.so /tmp/phb/*.o
python - <<'PY'
import ctypes, sys, os, numpy as np
sys.path.insert(0, os.getcwd())
import paper_2002_04989_b200._native as nat
lib = nat.load('/tmp/phb/libeigenid_b200.so')
from paper_2002_04989_b200.engine import random_symmetric
from paper_2002_04989_b200 import IdentityEngine
n = int(os.environ.get('N', '4096')); rows = int(os.environ.get('R', '147'))
a = random_symmetric(42, n) * np.sqrt(2.0 / n)
eng = IdentityEngine()
lam, mu = eng.minor_spectra(a, 0, rows)
buf = (ctypes.c_ulonglong * 16)()
lib.eigenid_debug_phase_cycles(buf)
names = ['other', 'copy', 'panel', 'band+VT', 'gemm1', 'Y,M,W2', 'gemm2', '-']
tot = sum(buf[i] for i in range(8))
print('stage 1 (CTA 0):')
for i in range(8): print(f'  {names[i]:10s} {buf[i]/1.965e9*1e3:9.2f} ms  {100*buf[i]/max(tot,1):5.1f}%')
b2 = (ctypes.c_ulonglong * 8)()
lib.eigenid_debug_bulge_cycles(b2)
names = ['loop/sweep', 'prefetch issue', 'right-apply+hh', 'left-apply+C store', 'wait D', 'two-sided+store', 'wait prev sweep']
tot = sum(b2[i] for i in range(7))
print('stage 2 (warp 0):')
for i in range(7): print(f'  {names[i]:20s} {b2[i]/1.965e9*1e3:9.2f} ms  {100*b2[i]/max(tot,1):5.1f}%')
PY
