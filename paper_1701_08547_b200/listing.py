"""Object-level disassembly parsing (the value API of occmix/sass.py).

The bulk path of this package never builds per-instruction Python objects:
``sass.tokenize`` turns a listing into K0's 4-byte records in C++.  This
module keeps the reference's *object* API for callers that want it --
``Instruction`` / ``Operand`` / ``OperandKind`` (ref sass.py:45-107),
``classify_operand`` (:60-77), ``render_instruction`` (:117-125),
``parse_instruction_line`` (:245-310) and ``parse_disassembly`` (:313-339)
-- with the same grammar, skip rules, quirks and error messages.  It is
host ingest, not per-candidate work.
"""

from __future__ import annotations

import enum
import re
from dataclasses import dataclass

from .errors import EmptyInputError, ParseError


class OperandKind(str, enum.Enum):
    REGISTER = "register"
    PREDICATE_REGISTER = "predicate-register"
    CONSTANT_BANK = "constant-bank"
    IMMEDIATE = "immediate"
    MEMORY = "memory"
    SPECIAL = "special"


# operand syntax, tested in the reference's order (sass.py:60-77)
_OPERAND_RULES = (
    (re.compile(r"R\d+(\.\w+)*$").match, OperandKind.REGISTER),
    (re.compile(r"c\[[^]]*\]\[[^]]*\]", re.IGNORECASE).match, OperandKind.CONSTANT_BANK),
    (lambda t: "[" in t, OperandKind.MEMORY),
    (re.compile(r"P\d+$").match, OperandKind.PREDICATE_REGISTER),
    (lambda t: t[:1].isdigit() or t.startswith(("0x", "-", "+")), OperandKind.IMMEDIATE),
)
_REG_NAME = re.compile(r"\bR\d+\b")


def classify_operand(token: str) -> OperandKind:
    for test, kind in _OPERAND_RULES:
        if test(token):
            return kind
    return OperandKind.SPECIAL


@dataclass(frozen=True)
class Operand:
    text: str
    kind: OperandKind

    @property
    def register_occurrences(self) -> int:
        return len(_REG_NAME.findall(self.text))


@dataclass(frozen=True)
class Instruction:
    opcode: str
    modifiers: tuple[str, ...] = ()
    operands: tuple[Operand, ...] = ()
    predicate: str | None = None
    address: int | None = None

    def __post_init__(self):
        if not self.opcode or not re.match(r"[A-Z][A-Z0-9]*$", self.opcode):
            raise ParseError(f"bad opcode {self.opcode!r}")

    @property
    def register_operand_count(self) -> int:
        return sum(op.register_occurrences for op in self.operands)

    def normalized(self) -> "Instruction":
        if self.address is None:
            return self
        return Instruction(self.opcode, self.modifiers, self.operands, self.predicate, None)


def render_instruction(instr: Instruction) -> str:
    head = ([instr.predicate] if instr.predicate else []) + \
        [instr.opcode + "".join(instr.modifiers)]
    if instr.operands:
        head.append(", ".join(op.text for op in instr.operands))
    return " ".join(head) + " ;"


# line grammar (sass.py:226-233)
_CTRL_PREFIX = re.compile(r"^\s*\[[-\w:]+\]")
_ADDRESS = re.compile(r"^\s*/\*\s*([0-9a-fA-F]+)\s*\*/")
_TAIL_COMMENT = re.compile(r"/\*.*?\*/\s*$")
_LABEL = re.compile(r"^\s*([A-Za-z_$][\w$.@]*)\s*:\s*$")
_GUARD = re.compile(r"^@!?P\w+$|^@!?PT$")
_OPCODE = re.compile(r"^([A-Z][A-Z0-9]*)((?:\.[^\s.]+)*)$")
_HEADERS = (re.compile(r"^\s*Function\s*:\s*(\S+)\s*$"),
            re.compile(r"^\s*\.section\s+\.text\.([^,\s]+)"))


def _strip_decorations(line: str) -> tuple[str, int | None]:
    """Drop the scheduling prefix, the address and trailing comments."""
    line = _CTRL_PREFIX.sub("", line, count=1)
    address = None
    m = _ADDRESS.match(line)
    if m:
        address = int(m.group(1), 16)
        line = line[m.end():]
    while True:
        shorter = _TAIL_COMMENT.sub("", line).rstrip()
        if shorter == line:
            break
        line = shorter
    return line.strip().strip("{}").strip(), address


def parse_instruction_line(line: str, lineno: int | None = None) -> Instruction | None:
    """One instruction, or None for a line that is not instruction-shaped."""
    body, address = _strip_decorations(line)
    if not body or body.startswith((".", "//", "/*")) or _LABEL.match(body):
        return None
    predicate = None
    first, _, rest = body.partition(" ")
    if _GUARD.match(first):
        predicate, body = first, rest.strip()
        if not body:
            raise ParseError("predicate guard with no instruction", lineno)
    token = body.split(None, 1)[0].rstrip(";")
    if not _OPCODE.match(token):
        return None
    if not body.rstrip().endswith(";"):
        raise ParseError(f"instruction {token!r} missing terminating ';'", lineno)
    head, _, operand_text = body.rstrip()[:-1].strip().partition(" ")
    m = _OPCODE.match(head)
    modifiers = tuple("." + part for part in m.group(2).split(".") if part)
    operands = tuple(Operand(t, classify_operand(t))
                     for t in (x.strip() for x in operand_text.split(",")) if t)
    return Instruction(m.group(1), modifiers, operands, predicate, address)


def _header(line: str) -> str | None:
    for rx in _HEADERS:
        m = rx.match(line)
        if m:
            return m.group(1)
    m = _LABEL.match(line)
    return m.group(1) if m else None


def parse_disassembly(text: str) -> list[tuple[str, list[Instruction]]]:
    """(function name, instructions) in file order (ref sass.py:313-339).
    A header repeating the current name continues that function; labels
    count as headers (the reference's documented behaviour)."""
    lines = text.splitlines()
    if not any(_header(ln) for ln in lines):
        raise EmptyInputError("no functions found")
    out: list[tuple[str, list[Instruction]]] = []
    name: str | None = None
    body: list[Instruction] = []
    for lineno, raw in enumerate(lines, start=1):
        h = _header(raw)
        if h is not None:
            if h != name:
                if name is not None:
                    out.append((name, body))
                name, body = h, []
            continue
        ins = parse_instruction_line(raw, lineno)
        if ins is None:
            continue
        if name is None:
            raise ParseError("instruction before any function header", lineno)
        body.append(ins)
    if name is not None:
        out.append((name, body))
    if not out:
        raise EmptyInputError("no functions found")
    return out
