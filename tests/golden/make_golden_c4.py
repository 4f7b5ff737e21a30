"""Generates tests/golden/reference_c4.npz: the UNMODIFIED reference on the
headline config C4 (n = 4096 GOE), sampled.

Input: random_symmetric(42, 4096).scaled(sqrt(2/4096)) (matrix_io.cpp:171-181,
matrix.cpp:82-86) built by the reference itself.  Outputs, all from
oracle/_ref/libeigenid_ref.so:
  * lam   — eigenvalues(A)                       (eigensolve.cpp:130-132)
  * mu    — eigenvalues(minor_matrix(j)) for the sampled j (identity.cpp:303-306)
  * rows  — out[j*n + i] for the sampled j, i.e. the reference's identity for
            those columns from the reference's own spectra (identity.cpp:308-314)
A full reference run is ~16 h on 8 cores; this sample takes about
10 minutes.  Build container only (needs /root/reference via oracle/_ref).

    python tests/golden/make_golden_c4.py
"""
import hashlib
import math
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import Reference  # noqa: E402

N = 4096
SEED = 42
JS = [0, 1, 2, 511, 1024, 1365, 2047, 2048, 2500, 3000, 3333, 3583, 4000, 4093, 4094, 4095]


def main():
    ref = Reference()
    a = ref.random_symmetric(SEED, N) * math.sqrt(2.0 / N)
    t = time.time()
    lam = ref.eigenvalues(a)
    print(f"eig(A) {time.time() - t:.1f} s", flush=True)
    t = time.time()
    mu = ref.minor_spectra(a, JS, workers=os.cpu_count() or 1)
    print(f"{len(JS)} minors {time.time() - t:.1f} s", flush=True)
    rows = ref.identity_rows(lam, mu, workers=os.cpu_count() or 1)
    # identity_rows evaluates component (i, r % n) — the column index only
    # enters the bounds check, so row r is |v_{i, JS[r]}|^2 for every i.
    np.savez_compressed(os.path.join(HERE, "reference_c4.npz"),
                        n=np.array([N]), seed=np.array([SEED]), js=np.array(JS),
                        a_sha256=np.frombuffer(hashlib.sha256(a.tobytes()).digest(),
                                               dtype=np.uint8),
                        lam=lam, mu=mu, rows=rows)
    print("wrote reference_c4.npz", flush=True)


if __name__ == "__main__":
    main()
