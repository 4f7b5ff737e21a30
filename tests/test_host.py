"""Host-side mirror of the reference API (no GPU): matrix construction,
minor remap and config / error mapping (matrix.cpp, identity.cpp:124-129,
errors.hpp)."""
import numpy as np
import pytest

import paper_2002_04989_b200 as eid
from paper_2002_04989_b200 import errors


def test_build_strict_rejects_asymmetric():
    with pytest.raises(eid.AsymmetricInput):
        eid.SymmetricMatrix.build(2, [1.0, 2.0, 3.0, 4.0])


def test_build_symmetrize_matches_reference_rule(oracle):
    g = oracle.gaussian_stream(9, 16).reshape(4, 4)
    m = eid.SymmetricMatrix.build(4, g, policy="symmetrize")
    want = oracle.random_symmetric(9, 4)  # random_symmetric = build(kSymmetrize)
    assert np.array_equal(m.array(), want)


def test_build_errors():
    with pytest.raises(eid.NonFiniteEntry):
        eid.SymmetricMatrix.build(1, [np.nan])
    with pytest.raises(eid.DimensionMismatch):
        eid.SymmetricMatrix.build(2, [1.0, 2.0, 3.0])
    with pytest.raises(eid.DimensionMismatch):
        eid.SymmetricMatrix.build(0, [])


def test_minor_matrix_remap(oracle):
    a = oracle.random_symmetric(3, 7)
    m = eid.SymmetricMatrix.build(7, a)
    for j in range(7):
        assert np.array_equal(m.minor_matrix(j).array(), oracle.minor(a, j))
    with pytest.raises(eid.IndexOutOfRange):
        m.minor_matrix(7)
    with pytest.raises(eid.MatrixTooSmall):
        eid.SymmetricMatrix.identity(1).minor_matrix(0)


def test_error_mapping():
    cases = {1: eid.MatrixTooSmall, 3: eid.ConvergenceFailure,
             4: eid.NonFiniteIntermediate, 5: eid.InternalInconsistency,
             6: eid.ConfigError, 7: eid.IndexOutOfRange, 20: eid.DeviceError,
             21: eid.DeviceError}
    for code, cls in cases.items():
        with pytest.raises(cls):
            errors.raise_for(code, "x")
    with pytest.raises(eid.DegenerateEigenvalue) as ei:
        errors.raise_for(2, "deg", gap=0.25)
    assert ei.value.gap() == 0.25
    errors.raise_for(0, "ok")  # no raise
    assert issubclass(eid.DegenerateEigenvalue, eid.Error)


def test_config_validation_before_device():
    with pytest.raises(eid.ConfigError):
        eid.IdentityEngine(eid.IdentityConfig(batch_size=0))
    with pytest.raises(eid.ConfigError):
        eid.IdentityEngine(eid.IdentityConfig(degeneracy_tol=-1.0))
