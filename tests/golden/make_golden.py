"""Generates tests/golden/*.npz from the UNMODIFIED reference.

Runs in the build container only (it needs oracle/_ref/libeigenid_ref.so,
compiled from /root/reference/proj/src by oracle/Makefile).  The outputs are
committed so the oracle restatement and the GPU path can be pinned against
the reference's own numbers on a box where /root/reference does not exist.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import OracleError, Reference  # noqa: E402


def main():
    ref = Reference()
    out = {}
    # seeded inputs + full pipeline (acceptance.cpp:54-73 sizes n = 2..64,
    # seeds 1000+t), several batch sizes and the log-domain evaluation
    cases = [(1000 + t, 2 + t % 63) for t in range(0, 100, 7)] + [(1, 64), (77, 100)]
    for seed, n in cases:
        a = ref.random_symmetric(seed, n)
        key = f"s{seed}_n{n}"
        out[f"{key}_a"] = a
        out[f"{key}_lam"] = ref.eigenvalues(a)
        out[f"{key}_all64"] = ref.all_magnitudes(a, batch=64, workers=1)
        if n <= 64:
            out[f"{key}_all1"] = ref.all_magnitudes(a, batch=1, workers=1)
            out[f"{key}_all8"] = ref.all_magnitudes(a, batch=8, workers=1)
            out[f"{key}_log"] = ref.all_magnitudes(a, batch=64, workers=1, log_domain=True)
        d, e = ref.tridiagonalize(a)
        out[f"{key}_d"], out[f"{key}_e"] = d, e
    out["cases"] = np.array(cases, dtype=np.int64)
    # uniform distribution input (matrix_io.cpp:46-51)
    out["uniform_s5_n9"] = ref.random_symmetric(5, 9, uniform=True)
    # hand cases (test_identity.cpp:216-227, :275-282)
    out["hand_2x2"] = ref.all_magnitudes(np.array([[2.0, 1.0], [1.0, 2.0]]), workers=1)
    out["hand_diag123"] = ref.all_magnitudes(np.diag([1.0, 2.0, 3.0]), workers=1)
    blk = np.array([[2.0, 1.0, 0.0], [1.0, 2.0, 0.0], [0.0, 0.0, 10.0]])
    try:
        out["hand_block"] = ref.all_magnitudes(blk, workers=1)
    except OracleError as e:  # recorded either way
        out["hand_block_err"] = np.array([e.code])
    # degenerate identity(5) -> DegenerateEigenvalue (test_identity.cpp:262-273)
    try:
        ref.all_magnitudes(np.eye(5), workers=1)
        out["deg_code"] = np.array([0])
    except OracleError as e:
        out["deg_code"] = np.array([e.code])
        out["deg_gap"] = np.array([e.gap])
    # overflow robustness (test_identity.cpp:284-296): n = 300, x1e3
    a = ref.random_symmetric(1, 300) * 1e3
    out["ovf_a_seed"] = np.array([1])
    out["ovf_all"] = ref.all_magnitudes(a, workers=0)
    # C5-style identity-only sample at n = 8192 (reference identity rows)
    from oracle.oracle import Oracle
    orc = Oracle()
    n = 8192
    lam = orc.c5_lambda(5, n)
    rows = [0, 4095, 8191]
    mu = orc.c5_mu_rows(5, lam, rows)
    out["c5_lam_8192"] = lam
    out["c5_rows"] = np.array(rows)
    out["c5_mu_8192"] = mu
    out["c5_id_8192"] = ref.identity_rows(lam, mu, workers=0)
    # sign recovery (signs.cpp:48-120): every eigenvector of small seeded
    # matrices, magnitudes and eigenvalues from the reference itself
    for n, seed in ((15, 8), (33, 21), (100, 77)):
        a = ref.random_symmetric(seed, n)
        lam = ref.eigenvalues(a)
        mags = ref.all_magnitudes(a, workers=1).reshape(n, n)
        out[f"signs_n{n}_a"] = a
        out[f"signs_n{n}_lam"] = lam
        out[f"signs_n{n}_mags"] = mags
        out[f"signs_n{n}_v"] = np.stack([ref.recover_signs(a, i, mags[:, i], lam[i])
                                         for i in range(n)])
    out["signs_hand_2x2"] = ref.recover_signs(np.array([[2.0, 1.0], [1.0, 2.0]]), 0,
                                              [0.5, 0.5], 1.0)
    out["signs_hand_diag"] = ref.recover_signs(np.diag([1.0, 2.0]), 1, [0.0, 1.0], 2.0)
    np.savez_compressed(os.path.join(HERE, "reference_golden.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
