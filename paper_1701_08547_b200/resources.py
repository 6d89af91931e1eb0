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


# ---------------------------------------------------------------------------
# ptxas -v resource report (restates occmix/sass.py:132-216)
# ---------------------------------------------------------------------------
# Grammar of the lines that matter (anything else is ignored):
#   ... Compiling entry function '<name>' [for 'sm_<digits>']   opens a stanza
#   ptxas info : Used <clause>, <clause>, ...                  resource clauses
#   ... <n> bytes spill stores / loads                         spill counters
# A clause is "<n> register(s)" or "<n> bytes (smem|lmem|gmem|stack frame|
# cmem[<bank>])"; anything else is a ParseError carrying the line number.
# 'sm_100a' does not match the optional target group (digits must be
# followed by the quote), so such stanzas get target_cc None, as in the
# reference.

_ENTRY = re.compile(r"Compiling entry function\s+'(?P<name>[^']+)'"
                    r"(?:\s+for\s+'sm_(?P<sm>\d+)')?")
_USED = re.compile(r"ptxas\s+info\s*:\s*Used\b(?P<rest>.*)$")
_CLAUSE_REGS = re.compile(r"^\s*(\d+)\s+registers?\s*$")
_CLAUSE_BYTES = re.compile(r"^\s*(\d+)\s+bytes\s+"
                           r"(?P<what>smem|lmem|gmem|stack frame|cmem\[(?P<bank>\d+)\])\s*$")
_SPILLS = re.compile(r"(\d+)\s+bytes\s+spill\s+(stores|loads)")


def _cc_of_sm(digits: str) -> float:
    v = int(digits)
    return (v // 10) + (v % 10) / 10.0


class _Stanza:
    __slots__ = ("name", "regs", "smem", "cmem", "spill_loads", "spill_stores", "cc")

    def __init__(self, name: str, cc):
        self.name, self.cc = name, cc
        self.regs = self.smem = self.spill_loads = self.spill_stores = 0
        self.cmem: list = []

    def done(self) -> KernelResources:
        return KernelResources(self.name, self.regs, self.smem, tuple(self.cmem),
                               self.spill_loads, self.spill_stores, self.cc)

    def used(self, rest: str, lineno: int):
        for clause in (c.strip() for c in rest.split(",")):
            if not clause:
                continue
            m = _CLAUSE_REGS.match(clause)
            if m:
                self.regs = int(m.group(1))
                continue
            m = _CLAUSE_BYTES.match(clause)
            if not m:
                raise ParseError(f"malformed resource clause {clause!r}", lineno)
            what = m.group("what")
            if what == "smem":
                self.smem = int(m.group(1))
            elif what.startswith("cmem"):
                self.cmem.append((int(m.group("bank")), int(m.group(1))))


def parse_resource_report(text: str) -> list[KernelResources]:
    """One KernelResources per 'Compiling entry function' stanza (ref
    sass.py:143-216).  EmptyInputError without any stanza."""
    from .errors import EmptyInputError
    out: list[KernelResources] = []
    cur: _Stanza | None = None
    for lineno, line in enumerate(text.splitlines(), start=1):
        m = _ENTRY.search(line)
        if m:
            if cur is not None:
                out.append(cur.done())
            cur = _Stanza(m.group("name"), _cc_of_sm(m.group("sm")) if m.group("sm") else None)
            continue
        if cur is None:
            continue
        m = _USED.search(line)
        if m:
            cur.used(m.group("rest"), lineno)
            continue
        for amount, kind in _SPILLS.findall(line):
            if kind == "loads":
                cur.spill_loads = int(amount)
            else:
                cur.spill_stores = int(amount)
    if cur is not None:
        out.append(cur.done())
    if not out:
        raise EmptyInputError("no kernel resource stanzas found")
    return out
