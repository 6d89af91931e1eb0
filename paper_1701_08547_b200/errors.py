"""Exception hierarchy of the public API (mirrors occmix/errors.py:4-48).

Every class keeps the reference's name, base class and constructor
arguments so ``except occmix.IllegalLaunchError`` style handlers keep
working when this package is swapped in.  The C ABI reports failures as
integer status codes (include/occx.h ``occx_status``); ``raise_status``
maps a code back onto the matching class.
"""

from __future__ import annotations


class StaticAnalysisError(Exception):
    """Root of every error this package raises (ref errors.py:4)."""


class ParseError(StaticAnalysisError):
    """Malformed text input; ``line`` is 1-based when known (ref errors.py:8-15)."""

    def __init__(self, message: str, line: int | None = None):
        self.line = line
        super().__init__(message if line is None else f"line {line}: {message}")


class EmptyInputError(ParseError):
    """Nothing recognizable in the input (ref errors.py:18)."""


class ArchSpecError(StaticAnalysisError):
    """An architecture descriptor breaks a hardware invariant (ref errors.py:22-27)."""

    def __init__(self, field: str, message: str):
        self.field = field
        super().__init__(f"{field}: {message}")


class UnknownArchitectureError(StaticAnalysisError):
    """Name not found in the architecture database (ref errors.py:30-36)."""

    def __init__(self, name: str, known: list[str]):
        self.name = name
        self.known = known
        super().__init__(f"unknown architecture {name!r}; known: {', '.join(known)}")


class UnsupportedArchitectureError(StaticAnalysisError):
    """No throughput-table column for this compute capability (ref errors.py:39)."""


class IllegalLaunchError(StaticAnalysisError):
    """Launch parameters the architecture cannot accept (ref errors.py:43)."""


class NoCandidatesError(StaticAnalysisError):
    """Pruning emptied the thread dimension (ref errors.py:47)."""


class DeviceError(StaticAnalysisError):
    """CUDA / NCCL / capacity failure inside the B200 backend (no reference
    counterpart: the reference never touches a device)."""


# occx_status codes (include/occx.h) -> exception class.
_STATUS_CLASS = {
    1: ValueError,
    2: IllegalLaunchError,
    3: UnsupportedArchitectureError,
    4: NoCandidatesError,
    5: ArchSpecError,
    6: DeviceError,
    7: DeviceError,
    8: DeviceError,
}


def raise_status(code: int, what: str) -> None:
    """Raise the exception class that corresponds to a non-zero occx_status."""
    if code == 0:
        return
    cls = _STATUS_CLASS.get(code, DeviceError)
    if cls is ArchSpecError:
        raise ArchSpecError("arch", what)
    raise cls(what)
