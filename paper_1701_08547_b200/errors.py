"""Exception hierarchy of the public API, and the C-ABI status mapping.

Class names, bases, constructor arguments and messages are those of
occmix/errors.py:4-48, so ``except occmix.IllegalLaunchError`` style
handlers keep working when this package is swapped in.  The C ABI reports
failures as integer ``occx_status`` codes (include/occx.h); each class
that a code maps onto carries it as ``status`` and ``raise_status`` turns
a code back into the exception.
"""

from __future__ import annotations


class StaticAnalysisError(Exception):
    """Root of every error this package raises (ref errors.py:4)."""

    status = 0


class ParseError(StaticAnalysisError):
    """Malformed text; ``line`` is the 1-based line when known (ref errors.py:8-15)."""

    def __init__(self, message: str, line: int | None = None):
        self.line = line
        if line is not None:
            message = f"line {line}: {message}"
        super().__init__(message)


class EmptyInputError(ParseError):
    """No stanza / function found in the input (ref errors.py:18)."""


class ArchSpecError(StaticAnalysisError):
    """Descriptor field ``field`` breaks a hardware invariant (ref errors.py:22-27)."""

    status = 5     # OCCX_ERR_ARCH_SPEC: rejected by occx_pack_arch / the kernels

    def __init__(self, field: str, message: str):
        self.field = field
        super().__init__(field + ": " + message)


class UnknownArchitectureError(StaticAnalysisError):
    """Name not in the user specs or the built-in table (ref errors.py:30-36)."""

    def __init__(self, name: str, known: list[str]):
        self.name, self.known = name, known
        super().__init__("unknown architecture %r; known: %s" % (name, ", ".join(known)))


class UnsupportedArchitectureError(StaticAnalysisError):
    """Compute capability without a throughput column (ref errors.py:39)."""

    status = 3     # OCCX_ERR_UNSUPPORTED_ARCH


class IllegalLaunchError(StaticAnalysisError):
    """Launch the architecture cannot accept (ref errors.py:43)."""

    status = 2     # OCCX_ERR_ILLEGAL_LAUNCH


class NoCandidatesError(StaticAnalysisError):
    """Static pruning left no thread count (ref errors.py:47)."""

    status = 4     # OCCX_ERR_NO_CANDIDATES


class DeviceError(StaticAnalysisError):
    """CUDA / NCCL / capacity failure inside the B200 backend.  No reference
    counterpart: occmix never touches a device."""

    status = 6     # OCCX_ERR_CUDA (7 = OCCX_ERR_NCCL, 8 = OCCX_ERR_CAPACITY)


_BY_STATUS = {c.status: c for c in (ArchSpecError, UnsupportedArchitectureError,
                                    IllegalLaunchError, NoCandidatesError, DeviceError)}
_BY_STATUS[1] = ValueError          # OCCX_ERR_VALUE


def raise_status(code: int, what: str) -> None:
    """Raise the exception for a non-zero occx_status; return on 0."""
    if not code:
        return
    cls = _BY_STATUS.get(code, DeviceError)
    raise ArchSpecError("arch", what) if cls is ArchSpecError else cls(what)
