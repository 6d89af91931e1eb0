"""Host ingest mirrors (listing.py, resources.py) against the reference:
the 4000 reference-recorded fuzz listings of sass_fuzz.json, the resource
reports recorded in report.json, and ports of occmix tests/test_sass.py
expectations.  CPU only."""

import pytest

from helpers import load_golden
from paper_1701_08547_b200 import (EmptyInputError, OperandKind, ParseError, parse_disassembly,
                                   parse_instruction_line, parse_resource_report,
                                   render_instruction, workloads)
from paper_1701_08547_b200.listing import classify_operand


def _summary(text):
    try:
        funcs = parse_disassembly(text)
    except (ParseError, EmptyInputError) as exc:
        return ["err", type(exc).__name__, exc.line, str(exc)]
    except Exception as exc:
        return ["err", type(exc).__name__, None, str(exc)]
    return ["ok", [[n, [[i.opcode, list(i.modifiers), i.predicate is not None,
                         i.register_operand_count] for i in ins]] for n, ins in funcs]]


def test_parse_disassembly_matches_reference_fuzz():
    g = load_golden("sass_fuzz.json")
    bad = [(i, c["text"]) for i, c in enumerate(g["cases"]) if _summary(c["text"]) != c["result"]]
    assert not bad, bad[:3]


def test_resource_reports_match_reference():
    g = load_golden("report.json")
    archs = workloads.all_archs()
    for run in g["corpus"]:
        a = archs[run["arch"]]
        dyn = 1024 if run["case"] == "space_scale_dyn" else 0
        text = workloads.corpus_resource_report(g["n_kernels"], run["seed"],
                                                a.max_regs_per_thread,
                                                a.shared_mem_per_block - dyn)
        got = [[x.entry_name, x.registers_per_thread, x.static_shared_mem,
                [list(b) for b in x.const_mem_banks], x.spill_loads, x.spill_stores, x.target_cc]
               for x in parse_resource_report(text)]
        assert got == run["result"]["resources"]


def test_resource_report_errors_match_reference():
    g = load_golden("report.json")
    for case in g["errors"]:
        want = case["result"]
        if want["error"] not in ("EmptyInputError", "ParseError"):
            continue
        with pytest.raises((EmptyInputError, ParseError)) as ei:
            parse_resource_report(case["resources"])
        assert type(ei.value).__name__ == want["error"]
        assert str(ei.value) == want["message"]


def test_atax_fixture_report_parses():
    g = load_golden("report.json")
    (res,) = parse_resource_report(g["atax"]["ptxas"])
    assert (res.entry_name, res.registers_per_thread, res.static_shared_mem,
            res.const_mem_banks, res.target_cc) == ("_Z4ataxPfS_S_i", 27, 0, ((0, 352),), 3.5)
    ((name, ins),) = parse_disassembly(g["atax"]["sass"])
    assert len(ins) == 33


# ported expectations of occmix tests/test_sass.py
@pytest.mark.parametrize("token,kind", [
    ("R0", OperandKind.REGISTER), ("R12.64", OperandKind.REGISTER),
    ("P0", OperandKind.PREDICATE_REGISTER), ("c[0x0][0x140]", OperandKind.CONSTANT_BANK),
    ("[R2+0x10]", OperandKind.MEMORY), ("0x3f800000", OperandKind.IMMEDIATE),
    ("-1", OperandKind.IMMEDIATE), ("SR_TID.X", OperandKind.SPECIAL), ("RZ", OperandKind.SPECIAL),
])
def test_operand_tagging(token, kind):
    assert classify_operand(token) is kind


def test_parse_lines_and_round_trip():
    i = parse_instruction_line("        /*0048*/                   FFMA R0, R2, R3, R0 ;  /* 0x5b */")
    assert (i.opcode, i.address, i.register_operand_count) == ("FFMA", 0x48, 4)
    b = parse_instruction_line("@!P0 BRA `(.L_1) ;")
    assert b.predicate == "@!P0" and b.opcode == "BRA"
    m = parse_instruction_line("LDG.E.64 R4, [R2+0x8] ;")
    assert m.modifiers == (".E", ".64") and m.operands[1].kind is OperandKind.MEMORY
    d = parse_instruction_line("[B------:R-:W-:-:S04] { IADD3 R1, R1, 0x1, RZ ; }")
    assert d.opcode == "IADD3"
    for skip in ("", "   ", ".headerflags", "// c", "/* c */", ".L_3:", "BB0_1:"):
        assert parse_instruction_line(skip) is None
    with pytest.raises(ParseError):
        parse_instruction_line("MOV R1, R2", 7)
    assert render_instruction(m) == "LDG.E.64 R4, [R2+0x8] ;"
    assert parse_instruction_line(render_instruction(i)) == i.normalized()
    with pytest.raises(EmptyInputError):
        parse_disassembly("MOV R1, R2 ;\n")
    with pytest.raises(ParseError):
        parse_disassembly("MOV R1, R2 ;\nFunction : k\n")
