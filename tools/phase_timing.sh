# Per-phase clock64 breakdown of stage 1 (CTA 0) and stage 2 (warp 0 of CTA 0)
# on a build with -DEIGENID_PHASE_TIMING (development aid, not the product).
set -e
cd $GRAFT_REPO_ROOT
mkdir -p /tmp/phb
for f in paper_2002_04989_b200/csrc/*.cu; do nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DEIGENID_PHASE_TIMING $VARIANT -Xcompiler -fPIC -c $f -o /tmp/phb/$(basename $f).o; done
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
names = ['other', 'copy', 'panel', 'band+VT', 'fused', 'Y,M,W2', 'gemm2', 'gemm1']
tot = sum(buf[i] for i in range(8))
g1 = min(rows + 1, int(os.environ.get('SLOTS', '296')))
print(f'stage 1 (summed over {g1} CTAs, shown per CTA):')
for i in range(8): print(f'  {names[i]:10s} {buf[i]/g1/1.965e9*1e3:9.2f} ms  {100*buf[i]/max(tot,1):5.1f}%')
names2 = ['gram P', 'chol+inv', 'row_transform x3', 'gram Q', 'check+chol+mul+inv', '-', 'LU+inv+T+V']
print('  chol_panel sub-phases:')
for i in range(7):
    if names2[i] != '-': print(f'    {names2[i]:20s} {buf[8+i]/g1/1.965e9*1e3:9.2f} ms')
print(f'  panel_qr fallbacks (all CTAs): {buf[15]}')
sp = (ctypes.c_ulonglong * 1536)()
lib.eigenid_debug_cta_span(sp)
g = min(rows + 1, int(os.environ.get('SLOTS', '296')))
st = np.array([sp[2 * b] for b in range(g)], dtype=np.float64)
sm = np.array([sp[1024 + b] for b in range(g)])
en = np.array([sp[2 * b + 1] for b in range(g)], dtype=np.float64)
t0 = st.min()
dur = (en - st) / 1e6
print(f'stage 1 CTA spans (ms): start max {(st.max()-t0)/1e6:.2f}  dur min {dur.min():.1f} '
      f'median {np.median(dur):.1f} max {dur.max():.1f}')
order = np.argsort(dur)
print('  fastest (cta, sm, ms):', [(int(b), int(sm[b]), round(float(dur[b]), 1)) for b in order[:6]])
print('  slowest (cta, sm, ms):', [(int(b), int(sm[b]), round(float(dur[b]), 1)) for b in order[-6:]])
hist = np.histogram(dur, bins=8)
print('  hist:', [int(x) for x in hist[0]], [round(float(x), 0) for x in hist[1]])
b2 = (ctypes.c_ulonglong * 8)()
lib.eigenid_debug_bulge_cycles(b2)
names = ['loop/sweep', 'prefetch issue', 'right-apply+hh', 'left-apply+C store', 'wait D', 'two-sided+store', 'wait prev sweep']
tot = sum(b2[i] for i in range(7))
print('stage 2 (warp 0):')
for i in range(7): print(f'  {names[i]:20s} {b2[i]/1.965e9*1e3:9.2f} ms  {100*b2[i]/max(tot,1):5.1f}%')
PY
