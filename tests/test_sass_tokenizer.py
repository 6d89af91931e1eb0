"""The native disassembly tokenizer (occx_sass_parse, host C++) against the
reference parser: 4000 fuzzed listings whose parse_disassembly() results
were recorded from the reference (tests/golden/make_golden.py `sass`), and
the config-3 corpus.  CPU only -- the tokenizer is host code."""

import numpy as np

import oracle
from helpers import load_golden
from paper_1701_08547_b200 import sass, workloads


def _summary(text, chunk_bytes=0):
    try:
        r = sass.tokenize(text, chunk_bytes)
    except Exception as exc:
        from paper_1701_08547_b200.errors import StaticAnalysisError
        return ["err", type(exc).__name__, getattr(exc, "line", None), str(exc)]
    out = []
    for k, name in enumerate(r.names):
        instrs = []
        for rec in r.records[int(r.offsets[k]):int(r.offsets[k + 1])]:
            op, mods = r.signatures[(int(rec) >> 1) & 0xFFFF]
            instrs.append([op, list(mods), bool(int(rec) & 1), (int(rec) >> 17) & 0xFF])
        out.append([name, instrs])
    return ["ok", out]


def test_fuzz_matches_reference_parser():
    g = load_golden("sass_fuzz.json")
    bad = []
    for i, case in enumerate(g["cases"]):
        got = _summary(case["text"])
        want = case["result"]
        if got[0] == "err" and want[0] == "err":
            # same exception class, line and message
            if got[1:] != want[1:]:
                bad.append((i, got, want))
        elif got != want:
            bad.append((i, got, want))
    assert not bad, bad[:3]
    assert sum(g["outcomes"].values()) == len(g["cases"])


def test_corpus_text_matches_generator_records():
    c = workloads.make_corpus(300)
    r = sass.tokenize(workloads.corpus_text(c))
    assert r.names == [f"kern_{k:06d}" for k in range(300)]
    np.testing.assert_array_equal(r.offsets, c.offsets)
    ops = workloads.corpus_opcodes()
    want_sig = [(ops[o], workloads.MOD_SUBSETS[s]) for o, s in zip(c.opcode, c.subset)]
    assert [r.signatures[(x >> 1) & 0xFFFF] for x in r.records] == want_sig
    rec = workloads.corpus_records(c)
    np.testing.assert_array_equal(r.records >> 17, rec >> 17)       # regops
    np.testing.assert_array_equal(r.records & 1, rec & 1)           # guard


def test_corpus_aggregate_golden_via_tokenizer():
    """tokenize -> C oracle aggregate == the reference's parse+aggregate."""
    g = load_golden("corpus.json")
    c = workloads.make_corpus(g["n_kernels"])
    r = sass.tokenize(workloads.corpus_text(c))
    counts, order, regs = oracle.aggregate_records(r.records, r.offsets, r.class_lut())
    names = oracle.pyref.CLASS_NAMES
    for k, (name, pairs, reg) in enumerate(g["kernels"]):
        assert r.names[k] == name
        assert [[names[cl], int(counts[k, cl])] for cl in order[k] if cl >= 0] == pairs
        assert int(regs[k]) == reg


def test_chunked_parse_equals_single_chunk():
    """Force tiny chunks (many threads): identical results and errors."""
    g = load_golden("sass_fuzz.json")
    texts = [c["text"] for c in g["cases"][:600]]
    big = "".join(texts)                     # concatenation crosses chunk cuts everywhere
    c = workloads.make_corpus(120)
    texts.append(workloads.corpus_text(c))
    texts.append(big)
    single = [_summary(t) for t in texts]
    multi = [_summary(t, 97) for t in texts]
    assert multi == single
    # signature ids too: first-occurrence order whatever the chunking
    ok = [t for t, r in zip(texts, single) if r[0] == "ok" and len(t) > 2000]
    assert len(ok) >= 2
    for t in ok:
        a, b = sass.tokenize(t), sass.tokenize(t, 97)
        assert a.signatures == b.signatures
        assert np.array_equal(a.records, b.records) and np.array_equal(a.offsets, b.offsets)


def test_utf8_views_of_the_listing():
    """tokenize() reads an ASCII str's own buffer, encodes other text as
    UTF-8 and text with lone surrogates with 'surrogatepass': the three give
    the same functions and records as the plain listing."""
    base = ("\tFunction : kern_a\n"
            "        /*0000*/                   MOV R1, c[0x0][0x28] ;   /* 0x1 */\n"
            "        /*0010*/              @P0  IADD3 R2, R3, R4, RZ ;   /* 0x2 */\n"
            "\tFunction : kern_b\n"
            "        /*0000*/                   EXIT ;   /* 0x3 */\n")
    want = _summary(base)
    assert want[0] == "ok" and [n for n, _ in want[1]] == ["kern_a", "kern_b"]
    uni = base.replace("/* 0x2 */", "/* 0x2 é☃ */")
    sur = base.replace("/* 0x2 */", "/* 0x2 \ud800 */")
    assert _summary(uni) == want
    assert _summary(sur) == want
    named = base.replace("kern_b", "kern_é")
    got = _summary(named)
    assert [n for n, _ in got[1]] == ["kern_a", "kern_é"] and got[1][0] == want[1][0]
