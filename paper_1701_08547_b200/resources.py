"""Kernel resource record (mirrors occmix/sass.py:26-42).

Only the value type lives here.  The ptxas/disassembly text parsers of
occmix/sass.py are host-side ingest outside the scored hot path
(SURVEY.md §2 row 8, §8(f) rank 1); callers keep using the reference
parsers and hand their ``KernelResources`` / ``Instruction`` objects to
this package unchanged (duck typed).
"""

from __future__ import annotations

import re
from dataclasses import dataclass

from .errors import ParseError


@dataclass(frozen=True)
class KernelResources:
    entry_name: str
    registers_per_thread: int = 0
    static_shared_mem: int = 0
    const_mem_banks: tuple[tuple[int, int], ...] = ()
    spill_loads: int = 0
    spill_stores: int = 0
    target_cc: float | None = None

    def __post_init__(self):
        if not self.entry_name:
            raise ParseError("kernel entry name must be non-empty")
        if self.registers_per_thread < 0 or self.static_shared_mem < 0:
            raise ParseError("resource counts must be non-negative")


# ``\bR\d+\b`` occurrences anywhere in an operand (ref sass.py:57, :84-88)
_REG_TOKEN = re.compile(r"\bR\d+\b")


def register_occurrences(operand_text: str) -> int:
    return len(_REG_TOKEN.findall(operand_text))


def register_operand_count(instr) -> int:
    """Register operands of an instruction object: uses the object's own
    ``register_operand_count`` when it has one (reference ``Instruction``),
    else counts over ``operands[*].text`` (ref sass.py:105-107)."""
    n = getattr(instr, "register_operand_count", None)
    if n is not None:
        return int(n)
    return sum(register_occurrences(getattr(op, "text", op))
               for op in getattr(instr, "operands", ()))
