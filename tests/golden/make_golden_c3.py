"""Generates tests/golden/reference_c3.npz: the UNMODIFIED reference on config
C3 (n = 1024, prescribed spectrum linspace(-1, 1)), sampled rows.

Input: oracle.c3_matrix(1024, seed 3) — SURVEY §8 d3's recipe in plain
deterministic loops (bit-identical to the product's eigenid_c3_matrix, so
the GPU box rebuilds the same bytes without /root/reference).  Outputs from
oracle/_ref/libeigenid_ref.so: lambda(A), the minor spectra of the sampled
j, and the reference's full all_magnitudes (identity.cpp:294-316) restricted
to the sampled rows j.  Build container only.

    python tests/golden/make_golden_c3.py
"""
import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import Oracle, Reference  # noqa: E402

N = 1024
SEED = 3
JS = sorted(set(list(range(0, N, 37)) + [1, 2, 511, 512, 1021, 1022, 1023]))


def main():
    ref = Reference()
    a = Oracle().c3_matrix(N, SEED)
    t = time.time()
    full = ref.all_magnitudes(a, workers=os.cpu_count() or 1)
    print(f"reference all_magnitudes n={N}: {time.time() - t:.1f} s", flush=True)
    lam = ref.eigenvalues(a)
    mu = ref.minor_spectra(a, JS, workers=os.cpu_count() or 1)
    np.savez_compressed(os.path.join(HERE, "reference_c3.npz"),
                        n=np.array([N]), seed=np.array([SEED]), js=np.array(JS),
                        a_sha256=np.frombuffer(hashlib.sha256(a.tobytes()).digest(),
                                               dtype=np.uint8),
                        lam=lam, mu=mu, rows=full[JS],
                        col_sums=full.sum(axis=0), row_sums=full.sum(axis=1))
    print("wrote reference_c3.npz", flush=True)


if __name__ == "__main__":
    main()
