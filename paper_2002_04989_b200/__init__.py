"""B200-native eigenvector–eigenvalue identity (arxiv 2002.04989).

Drop-in for the reference hot path IdentityEngine::all_magnitudes
(proj/src/identity.cpp:294-316) and the eigenvalue solver beneath it.  The
computation runs in hand-written sm_100a kernels behind the C-ABI in
include/eigenid_b200.h; this package is the Python mirror of the reference's
C++ API over that boundary.
"""
from .errors import (AsymmetricInput, ConfigError, ConvergenceFailure,  # noqa: F401
                     DegenerateEigenvalue, DeviceError, DimensionMismatch, Error,
                     IndexOutOfRange, InternalInconsistency, MatrixTooSmall,
                     NonFiniteEntry, NonFiniteIntermediate, SignRecoveryFailure)
from .engine import (Device, IdentityConfig, IdentityEngine,  # noqa: F401
                     SymmetricMatrix, c3_matrix, eigenvalues, random_symmetric,
                     recover_signs)

__all__ = [
    "IdentityEngine", "IdentityConfig", "SymmetricMatrix", "eigenvalues", "Device",
    "random_symmetric", "recover_signs", "c3_matrix",
    "Error", "MatrixTooSmall", "DegenerateEigenvalue", "ConvergenceFailure",
    "NonFiniteIntermediate", "InternalInconsistency", "ConfigError",
    "IndexOutOfRange", "DeviceError", "AsymmetricInput", "NonFiniteEntry",
    "DimensionMismatch", "SignRecoveryFailure",
]
