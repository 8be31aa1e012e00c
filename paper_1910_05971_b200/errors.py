"""Error taxonomy of the drop-in, mirroring svcc.errors
(/root/reference/pkg/src/svcc/errors.py:4-19) name for name, plus the mapping
from the C-ABI status codes (include/fastsv.h)."""


class SvccError(Exception):
    """Base class for errors raised by this package."""


class InputError(SvccError):
    """Bad user input (out-of-range edge, negative vertex count, ...)."""


class VerificationError(SvccError):
    """A computed labeling disagrees with the oracle."""


class InvariantError(SvccError):
    """An algorithm invariant was violated (monotonicity, star at exit)."""


class DeviceError(SvccError, RuntimeError):
    """CUDA / NCCL runtime failure (status FSV_ERR_RUNTIME). Not in the
    reference, which never leaves the CPU."""


def raise_for_status(code: int, message: str) -> None:
    """Map a C-ABI status code to the reference exception classes."""
    if code == 0:
        return
    if code == 1:
        raise InputError(message)
    if code == 2:
        raise ValueError(message)
    if code == 3:
        raise InvariantError(message)
    raise DeviceError(message)
