"""Pin the oracle (oracle/pyref.py, oracle/occx_oracle.c) to the reference.

Every fixture in tests/golden/ was produced by tests/golden/make_golden.py
calling the reference occmix package itself.  CPU only.
"""


import numpy as np
import pytest

import oracle
from oracle import pyref
from paper_1701_08547_b200 import workloads
from helpers import problem_of, same_sum_semantics, spaces_of


def _grid_occ(archs, ai, mode, T, R, S):
    n = len(T)
    return oracle.occupancy_many(archs, np.full(n, ai), T, R, S, verbatim=bool(mode))


@pytest.mark.parametrize("ai", range(5))
@pytest.mark.parametrize("mode", [0, 1])
def test_c_oracle_limit_tables_exhaustive(golden, archs, ai, mode):
    """limit_by_warps / _registers / _smem over their full domains."""
    g = golden("occupancy_tables.npz")
    A = archs[ai]
    # warps (T 1..1100) and registers (T x R 0..300): S=0 keeps ls = Bmp
    T = np.repeat(np.arange(1, 1101), 301)
    R = np.tile(np.arange(301), 1100)
    o = _grid_occ(archs, ai, mode, T, R, np.zeros_like(T))
    legal = o["status"] == 0
    lw = np.where(legal, o["lw"], -1).reshape(1100, 301)[:, 0]
    lr = np.where(legal, o["lr"], -1).reshape(1100, 301)
    np.testing.assert_array_equal(lw, g[f"lw_{ai}_{mode}"])
    np.testing.assert_array_equal(lr, g[f"lr_{ai}_{mode}"])
    np.testing.assert_array_equal(o["rwl"].reshape(1100, 301)[0], g[f"rwl_{ai}_{mode}"])
    S = np.arange(A.shared_mem_per_block + 65)
    o = _grid_occ(archs, ai, mode, np.full_like(S, A.warp_size), np.zeros_like(S), S)
    np.testing.assert_array_equal(o["ls"], g[f"ls_{ai}_{mode}"])


def test_c_oracle_random_occupancy(golden, archs):
    rows = golden("occupancy_random.npz")["rows"]
    for mode in (0, 1):
        sel = rows[rows[:, 1] == mode]
        o = oracle.occupancy_many(archs, sel[:, 0], sel[:, 2], sel[:, 3], sel[:, 4],
                                  verbatim=bool(mode))
        illegal = sel[:, 5] == 1
        np.testing.assert_array_equal(o["status"] != 0, illegal)
        ok = ~illegal
        got = np.stack([o["wpb"], o["lw"], o["lr"], o["ls"], o["blocks"], o["aw"],
                        o["limiter"], o["occ"].view(np.int64)], 1)[ok]
        np.testing.assert_array_equal(got, sel[ok][:, 6:14])


def test_pyref_random_occupancy(golden, archs):
    rows = golden("occupancy_random.npz")["rows"][:20000]
    names = ("warps", "registers", "shared-memory", "illegal")
    for ai, mode, t, r, s, ill, *rest in rows.tolist():
        try:
            res = pyref.occupancy(archs[ai], t, r, s, bool(mode))
        except pyref.OracleIllegalLaunch:
            assert ill == 1
            continue
        assert ill == 0
        wpb, lw, lr, ls, b, aw, occ, lim = res
        assert [wpb, lw, lr, ls, b, aw, names.index(lim)] == rest[:7]
        assert np.float64(occ).view(np.int64) == rest[7]


def test_pyref_suggest(golden, archs):
    for row in golden("suggest.json")["rows"]:
        ai, mi, regs, smem, status = row[:5]
        try:
            s = pyref.suggest(archs[ai], regs, smem, bool(mi))
        except pyref.OracleIllegalLaunch:
            assert status == "illegal"
            continue
        assert status == "ok"
        assert [list(s["thread_candidates"]), s["register_headroom"], s["smem_budget"],
                s["best_occupancy"].hex(), s["best_threads"], s["best_blocks"]] == row[5:]


def test_thread_candidate_goldens(archs):
    # test_occupancy.py:163-168 + the sm_100 INI table
    assert [pyref.thread_candidates(a) for a in archs] == [
        (192, 256, 384, 512, 768), (128, 256, 512, 1024), (64, 128, 256, 512, 1024),
        (64, 128, 256, 512, 1024), (64, 128, 256, 512, 1024)]


def _pyref_counts(pairs):
    return {c: n for c, n in pairs}


def test_pyref_mix_features(golden):
    g = golden("mix.json")
    if not same_sum_semantics(g["meta"]):
        pytest.skip("goldens captured under a different CPython sum()")
    for v in g["variants"] + [dict(g["atax"])]:
        counts = _pyref_counts(v["counts"])
        assert pyref.intensity(counts).hex() == v["intensity"]
        for cc, f in v["features"].items():
            cc = float(cc)
            if f == "unsupported":
                with pytest.raises(pyref.OracleUnsupported):
                    pyref.cost_estimate(counts, v["reg_operands"], cc)
                continue
            assert pyref.cost_estimate(counts, v["reg_operands"], cc).hex() == f["cost"]
            assert [x.hex() for x in pyref.category_cycles(counts, v["reg_operands"],
                                                           cc).values()] == f["cycles"]
            assert [x.hex() for x in pyref.pipeline_utilization(
                counts, v["reg_operands"], cc).values()] == f["shares"]
            assert {k: x.hex() for k, x in pyref.per_class_cycles(
                counts, v["reg_operands"], cc).items()} == f["per_class"]
    for v in g["random"]:
        counts = _pyref_counts(v["counts"])
        scale = float.fromhex(v["scale"])
        assert pyref.cost_estimate(counts, v["reg_operands"], v["cc"], scale).hex() == \
            v["cost_scaled"]
        assert pyref.intensity(counts).hex() == v["intensity"]


def test_atax_mix_matches_workload(golden):
    """workloads.BASE_MIXES['atax'] is the reference's aggregate of the fixture."""
    a = golden("mix.json")["atax"]
    counts, regs, r = workloads.BASE_MIXES["atax"]
    assert [[c.value, n] for c, n in counts] == a["counts"]
    assert regs == a["reg_operands"]
    assert (a["flops"], a["mem"], a["ctrl"], a["total"]) == (17, 5, 11, 33)
    assert float.fromhex(a["intensity"]) == 3.4
    # the oracle's aggregate of the fixture's instruction stream
    table = {k: v.value for k, v in __import__(
        "paper_1701_08547_b200.mix", fromlist=["x"]).DEFAULT_OPCLASSES.items()}
    instrs = [(op, tuple(m), p is not None, n) for op, m, p, n in a["instructions"]]
    c, regs2 = pyref.aggregate(instrs, table)
    assert [[k, n] for k, n in c.items()] == a["counts"] and regs2 == regs


def test_c_oracle_corpus_aggregate(golden):
    g = golden("corpus.json")
    c = workloads.make_corpus(g["n_kernels"])
    import hashlib
    assert hashlib.sha256(workloads.corpus_text(c).encode()).hexdigest() == g["text_sha256"]
    counts, order, regs = oracle.aggregate_records(
        workloads.corpus_records(c), c.offsets, workloads.corpus_signature_lut())
    names = pyref.CLASS_NAMES
    for kk, (name, pairs, reg) in enumerate(g["kernels"]):
        got = [[names[cl], int(counts[kk, cl])] for cl in order[kk] if cl >= 0]
        assert got == pairs, name
        assert int(regs[kk]) == reg


@pytest.mark.parametrize("name", ["config1", "config2", "config4"])
def test_c_oracle_topk(golden, name):
    g = golden(f"topk_{name}.json")
    cfg = workloads.CONFIGS[name]()
    for mode in ("corrected", "verbatim"):
        if mode not in g:
            continue
        prob = problem_of(cfg, verbatim=(mode == "verbatim"))
        got = oracle.score_spaces(prob, spaces_of(cfg), threads=8)
        assert got.tolist() == g[mode], (name, mode)


def test_pyref_topk_config1(golden):
    g = golden("topk_config1.json")
    cfg = workloads.config1()
    prob = problem_of(cfg)
    cands = [(0, 0, t, 27, 0) for t in range(32, 1025, 32)]
    assert pyref.score_candidates(prob, cands) == g["corrected"]
    # top-16 thread counts of config 1
    top = [pyref.key_index(k) for k in g["corrected"][0]]
    assert [32 * (i + 1) for i in top] == [128, 256, 512, 1024, 224, 288, 672, 992, 160,
                                           192, 320, 384, 480, 640, 960, 928]


def test_pyref_naive_sum_semantics(golden):
    """CPython <= 3.11 sum() (the reference's recorded run, Python 3.10.12,
    /root/reference/pkg/test_output.txt:2): pyref under sum_semantics("naive")
    equals an independent left-to-right float64 accumulation (np.cumsum)
    of the same terms, and differs from this interpreter's compensated
    sum() on some sm35 mixes (so the mode is observable)."""
    import sys
    g = golden("mix.json")
    differ = 0
    for v in g["random"]:
        counts = dict(v["counts"])
        regs, cc, scale = v["reg_operands"], v["cc"], float.fromhex(v["scale"])
        col = pyref.column(cc)
        fl = [n * pyref.cpi(c, col) for c, n in counts.items() if pyref.CATEGORY.get(c) == "FLOPS"]
        nfl = pyref.flops(counts)
        coef = np.cumsum(fl)[-1] / nfl if nfl else pyref.cpi("FPIns32", col)
        terms = [coef * nfl, pyref.cpi("LdStIns", col) * pyref.mem(counts),
                 pyref.cpi("CtrlIns", col) * pyref.ctrl(counts), pyref.cpi("Regs", col) * regs]
        want = scale * float(np.cumsum(terms)[-1])
        with pyref.sum_semantics("naive"):
            got = pyref.cost_estimate(counts, regs, cc, scale)
        assert got.hex() == want.hex()
        differ += got != pyref.cost_estimate(counts, regs, cc, scale)
    if sys.version_info >= (3, 12):
        assert differ > 0, "naive and compensated sum() never differ on the golden mixes"
