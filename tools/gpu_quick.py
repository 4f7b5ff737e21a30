import sys, time, numpy as np
import os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.oracle import Oracle
from paper_2002_04989_b200 import IdentityEngine, IdentityConfig, eigenvalues
o = Oracle()
eng = IdentityEngine()
def rel(g, c):
    return float(np.max(np.abs(g - c) / (np.abs(c) * 1e-9 + 1e-12)))
for n in [2, 3, 5, 8, 16, 33, 64, 65, 80, 100, 130, 200, 300]:
    a = o.random_symmetric(1000 + n, n)
    t = time.time()
    try:
        g, lam, mu = eng.all_magnitudes(a, return_spectra=True)
    except Exception as ex:
        print(n, 'GPU EXC', ex); continue
    tg = time.time() - t
    c, lc, mc = o.all_magnitudes(a, return_spectra=True)
    g = g.reshape(n, n)
    print(n, 'lam maxabs', np.max(np.abs(lam - lc)), 'mu maxabs', np.max(np.abs(mu - mc)),
          'out maxabs', np.max(np.abs(g - c)), 'pred', rel(g, c), 'tg', round(tg, 4), flush=True)
    # identity-only bit exactness
    gi = eng.identity(lc, mc)
    print('   identity bit-exact:', bool((gi.view(np.uint64) == c.view(np.uint64)).all()))
for n in [2, 5, 64, 100, 257]:
    a = o.random_symmetric(7, n)
    ev = eigenvalues(a); evc = o.eigenvalues(a)
    print('eig', n, np.max(np.abs(ev - evc)))
# batched C2-like
A = np.stack([o.random_symmetric(b, 32) for b in range(64)])
G = eng.all_magnitudes_batched(A)
err = max(np.max(np.abs(G[b] - o.all_magnitudes(A[b]).reshape(-1))) for b in range(64))
print('batched maxabs', err)
