import os, sys, time, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ['EIGENID_PROFILE'] = '1'
from oracle.oracle import Oracle
from paper_2002_04989_b200 import IdentityEngine
o = Oracle(); eng = IdentityEngine()
for n in [int(x) for x in sys.argv[1:]]:
    a = o.random_symmetric(42, n) * np.sqrt(2.0 / n)
    for rep in range(2):
        t = time.time()
        g, lam, mu = eng.all_magnitudes(a, return_spectra=True)
        dt = time.time() - t
        g = g.reshape(n, n)
        print(f'n={n} rep={rep} wall={dt:.3f}s rowsum={np.max(np.abs(g.sum(1)-1)):.2e} colsum={np.max(np.abs(g.sum(0)-1)):.2e}', flush=True)
    lref = np.linalg.eigvalsh(a)
    print('  lam vs LAPACK', np.max(np.abs(lam - lref)))
    for j in [0, n // 2]:
        keep = np.r_[0:j, j + 1:n]
        mref = np.linalg.eigvalsh(a[np.ix_(keep, keep)])
        print('  mu', j, 'vs LAPACK', np.max(np.abs(mu[j] - mref)))
