"""The CPU oracle is pinned to the reference (CPU, no GPU needed).

* bit-exact against the committed golden vectors produced by the unmodified
  reference (tests/golden/make_golden.py), and
* bit-exact against oracle/_ref itself on fresh seeded inputs when it is
  built (this container),
* plus the reference's own known-answer tests (test_identity.cpp,
  acceptance.cpp) replayed on the oracle.
"""
import os

import numpy as np
import pytest

from oracle.oracle import OracleError

GOLD = os.path.join(os.path.dirname(__file__), "golden", "reference_golden.npz")


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


def bits(x):
    return np.ascontiguousarray(x, np.float64).view(np.uint64)


def test_seeded_inputs_match_reference_generator(oracle, gold):
    for seed, n in gold["cases"]:
        a = oracle.random_symmetric(int(seed), int(n))
        assert np.array_equal(bits(a), bits(gold[f"s{seed}_n{n}_a"])), (seed, n)
    u = oracle.random_symmetric(5, 9, uniform=True)
    assert np.array_equal(bits(u), bits(gold["uniform_s5_n9"]))


def test_pipeline_bit_exact_against_golden(oracle, gold):
    for seed, n in gold["cases"]:
        key = f"s{seed}_n{n}"
        a = gold[f"{key}_a"]
        d, e = oracle.tridiagonalize(a)
        assert np.array_equal(bits(d), bits(gold[f"{key}_d"]))
        assert np.array_equal(bits(e), bits(gold[f"{key}_e"]))
        assert np.array_equal(bits(oracle.eigenvalues(a)), bits(gold[f"{key}_lam"]))
        got = oracle.all_magnitudes(a, batch=64, threads=2)
        assert np.array_equal(bits(got), bits(gold[f"{key}_all64"])), key
        if n <= 64:
            for b in (1, 8):
                assert np.array_equal(bits(oracle.all_magnitudes(a, batch=b, threads=2)),
                                      bits(gold[f"{key}_all{b}"])), (key, b)
            # log-domain uses libm log/exp: same library on both sides
            assert np.array_equal(bits(oracle.all_magnitudes(a, log_domain=True, threads=2)),
                                  bits(gold[f"{key}_log"])), key


def test_hand_cases(oracle, gold):
    assert np.allclose(oracle.all_magnitudes(np.array([[2.0, 1.0], [1.0, 2.0]])), 0.5,
                       atol=1e-12, rtol=0)
    assert np.array_equal(oracle.all_magnitudes(np.array([[2.0, 1.0], [1.0, 2.0]])),
                          gold["hand_2x2"])
    d = oracle.all_magnitudes(np.diag([1.0, 2.0, 3.0]))
    assert np.allclose(d, np.eye(3), atol=1e-12)
    assert np.array_equal(d, gold["hand_diag123"])
    blk = np.array([[2.0, 1.0, 0.0], [1.0, 2.0, 0.0], [0.0, 0.0, 10.0]])
    assert np.array_equal(oracle.all_magnitudes(blk), gold["hand_block"])
    assert oracle.all_magnitudes(blk)[2, 0] <= 1e-8  # interlacing coincidence -> 0


def test_degenerate_raises_with_gap(oracle, gold):
    with pytest.raises(OracleError) as ei:
        oracle.all_magnitudes(np.eye(5))
    assert ei.value.code == int(gold["deg_code"][0]) == 2
    assert ei.value.gap == float(gold["deg_gap"][0])


def test_too_small(oracle):
    with pytest.raises(OracleError) as ei:
        oracle.all_magnitudes(np.eye(1))
    assert ei.value.code == 1


def test_overflow_case_matches_reference(oracle, gold):
    a = oracle.random_symmetric(1, 300) * 1e3
    got = oracle.all_magnitudes(a)
    assert np.all(np.isfinite(got))
    assert np.array_equal(bits(got), bits(gold["ovf_all"]))


def test_identity_stage_on_c5_sample(oracle, gold):
    lam = gold["c5_lam_8192"]
    assert np.array_equal(bits(oracle.c5_lambda(5, 8192)), bits(lam))
    mu = oracle.c5_mu_rows(5, lam, gold["c5_rows"])
    assert np.array_equal(bits(mu), bits(gold["c5_mu_8192"]))
    # interlacing by construction
    assert np.all(mu > lam[None, :-1]) and np.all(mu < lam[None, 1:])
    got = oracle.identity_rows(lam, mu)
    assert np.array_equal(bits(got), bits(gold["c5_id_8192"]))
    # column-of-|v|^2 sums to one for any interlacing mu (Lagrange identity)
    assert np.allclose(got.sum(axis=1), 1.0, atol=1e-11)


def test_sorted_pairing_is_a_reversal(oracle):
    """sorting both factor lists equals reversing them, which is
    what lets the GPU kernels skip the per-(i,j) sorts."""
    a = oracle.random_symmetric(3, 40)
    out, lam, mu = oracle.all_magnitudes(a, return_spectra=True)
    n = 40
    for j in (0, 17, 39):
        for i in (0, 5, 39):
            num = lam[i] - mu[j]
            den = np.array([lam[i] - lam[k] for k in range(n) if k != i])
            assert np.array_equal(np.sort(num), num[::-1])
            assert np.array_equal(np.sort(den), den[::-1])


def test_matches_reference_live(oracle, reference):
    for seed, n in ((7, 2), (8, 13), (9, 64), (10, 97)):
        a = reference.random_symmetric(seed, n)
        assert np.array_equal(bits(oracle.all_magnitudes(a)),
                              bits(reference.all_magnitudes(a, workers=2)))
        assert reference.last_solves == n + 1  # solve-count contract


def test_jacobi_equivalence(oracle, reference):
    """acceptance.cpp:54-73 on a subset: all_magnitudes vs the Jacobi oracle."""
    worst = 0.0
    for t in range(0, 100, 9):
        n = 2 + t % 63
        a = oracle.random_symmetric(1000 + t, n)
        m = oracle.all_magnitudes(a)
        _, vec = reference.jacobi(a)
        worst = max(worst, float(np.max(np.abs(m - vec ** 2))))
    assert worst <= 1e-8


def test_doubly_stochastic(oracle):
    m = oracle.all_magnitudes(oracle.random_symmetric(77, 100))
    assert np.max(np.abs(m.sum(0) - 1)) <= 1e-8
    assert np.max(np.abs(m.sum(1) - 1)) <= 1e-8


# ---------------------------------------------------------------- signs (f4)
def test_recover_signs_golden(oracle, gold):
    """signs.cpp:48-120 restated: every eigenvector of three seeded matrices
    bit-identical to the reference's recover_signs (golden vectors)."""
    for n in (15, 33, 100):
        a, lam, mags = gold[f"signs_n{n}_a"], gold[f"signs_n{n}_lam"], gold[f"signs_n{n}_mags"]
        want = gold[f"signs_n{n}_v"]
        for i in range(n):
            got = oracle.recover_signs(a, i, mags[:, i], lam[i])
            assert np.array_equal(got.view(np.uint64), want[i].view(np.uint64)), (n, i)


def test_recover_signs_hand_cases_and_errors(oracle, gold):
    """test_identity.cpp:313-354 known answers and error behaviour."""
    v = oracle.recover_signs(np.array([[2.0, 1.0], [1.0, 2.0]]), 0, [0.5, 0.5], 1.0)
    assert np.array_equal(v, gold["signs_hand_2x2"])
    assert abs(v[0] - 2 ** -0.5) < 1e-12 and abs(v[1] + 2 ** -0.5) < 1e-12
    v = oracle.recover_signs(np.diag([1.0, 2.0]), 1, [0.0, 1.0], 2.0)
    assert np.array_equal(v, gold["signs_hand_diag"])
    a = oracle.random_symmetric(8, 10)
    with pytest.raises(OracleError) as e:
        oracle.recover_signs(a, 0, np.full(10, 0.1), 123.0)
    assert e.value.code == 8  # SignRecoveryFailure
    with pytest.raises(OracleError) as e:
        oracle.recover_signs(a, 0, np.full(9, 0.1), 123.0)
    assert e.value.code == 9  # DimensionMismatch


def test_recover_signs_matches_reference_live(oracle, reference):
    for n, seed in ((5, 3), (40, 4), (64, 5)):
        a = reference.random_symmetric(seed, n)
        lam = reference.eigenvalues(a)
        mags = reference.all_magnitudes(a, workers=1).reshape(n, n)
        for i in range(0, n, 3):
            want = reference.recover_signs(a, i, mags[:, i], lam[i])
            got = oracle.recover_signs(a, i, mags[:, i], lam[i])
            assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
