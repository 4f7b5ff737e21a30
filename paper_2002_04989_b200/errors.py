"""Typed errors mirroring proj/include/eigenid/errors.hpp:11-107.

The C-ABI returns integer status codes (include/eigenid_b200.h); `raise_for`
turns them into the same exception hierarchy the reference throws, plus
DeviceError for CUDA failures (there is no CPU fallback).
"""


class Error(RuntimeError):
    """eigenid::Error (errors.hpp:11-14)."""


class AsymmetricInput(Error):
    pass


class NonFiniteEntry(Error):
    pass


class IndexOutOfRange(Error):
    pass


class MatrixTooSmall(Error):
    pass


class DimensionMismatch(Error):
    pass


class ConvergenceFailure(Error):
    pass


class DegenerateEigenvalue(Error):
    """errors.hpp:58-66 — carries the offending gap."""

    def __init__(self, msg: str, gap: float):
        super().__init__(msg)
        self._gap = gap

    def gap(self) -> float:
        return self._gap


class NonFiniteIntermediate(Error):
    pass


class InternalInconsistency(Error):
    pass


class ConfigError(Error):
    pass


class SignRecoveryFailure(Error):
    """errors.hpp:79-82 (recover_signs)."""


class DeviceError(Error):
    """New: a CUDA failure or a missing device (no CPU fallback)."""

    def __init__(self, msg: str, cuda_error: int = 0):
        super().__init__(msg)
        self.cuda_error = cuda_error


OK = 0
_CODES = {
    1: MatrixTooSmall,
    3: ConvergenceFailure,
    4: NonFiniteIntermediate,
    5: InternalInconsistency,
    6: ConfigError,
    7: IndexOutOfRange,
    8: SignRecoveryFailure,
    9: DimensionMismatch,
    10: NonFiniteEntry,
    11: AsymmetricInput,
}


def raise_for(code: int, msg: str, gap: float = 0.0, cuda_error: int = 0):
    if code == OK:
        return
    if code == 2:
        raise DegenerateEigenvalue(msg, gap)
    if code in _CODES:
        raise _CODES[code](msg)
    raise DeviceError(msg, cuda_error)
