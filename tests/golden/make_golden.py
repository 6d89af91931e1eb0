"""Generate the golden fixtures in tests/golden/ FROM THE REFERENCE ITSELF.

Run in the build container (the reference is not on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py [--big]

Imports occmix read-only from /root/reference/pkg/src and records, tagged
with sys.version (CPython's float sum() changed in 3.12):
  occupancy_tables.npz   exhaustive limit tables (5 archs x 2 modes):
                         limit_by_warps T 1..1100, limit_by_registers T x R
                         (T 1..1100, R 0..300), limit_by_smem S 0..Smax+64
  occupancy_random.npz   200k random occupancy() calls, every field
  suggest.json           suggest() over archs x regs x smem x modes
  partial_table.json     cost / cycles / shares / per_class outcomes (hex or
                         KeyError) under partial throughput tables
  mix.json               ATAX fixture aggregate, workload variant features,
                         3000 random mixes (cost/intensity/shares as hex)
  corpus.json            aggregate() of the reference parser over the first
                         2000 kernels of the config-3 corpus text
  specs.json             parse_space_file / parse_arch_config / parse_opclass_table
                         outcomes (values or error class, line, message) on
                         fuzzed spec texts
  topk_config{1,2,4}.json (and 5 with --big): per-segment top-16 keys of
                         the scoring composition, computed from reference
                         functions (limit tables, static/rule_prune,
                         cost_estimate, intensity)
The workload *inputs* come from paper_1701_08547_b200.workloads.
"""

from __future__ import annotations

import hashlib
import json
import math
import os
import random
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, REF)
sys.dont_write_bytecode = True

import occmix as R  # noqa: E402  (the reference)
from occmix import mix as Rmix  # noqa: E402
Rocc = sys.modules["occmix.occupancy"]

from paper_1701_08547_b200 import workloads as W  # noqa: E402


def ref_arch(spec):
    """Reference ArchSpec with the same field values."""
    if spec.family.value in ("fermi", "kepler", "maxwell", "pascal") and \
            spec.name == R.builtin_arch(spec.family.value).name:
        return R.builtin_arch(spec.family.value)
    return R.arch.parse_arch_config(W.SM100_INI)[0]


ARCHS = [ref_arch(a) for a in W.all_archs()]
MODES = (R.Mode.CORRECTED, R.Mode.VERBATIM)
META = {"python": sys.version.split()[0], "sum": "neumaier" if sys.version_info >= (3, 12)
        else "naive", "generator": "tests/golden/make_golden.py"}


def _call(f, *a):
    try:
        return f(*a)
    except R.IllegalLaunchError:
        return -1


def occupancy_tables():
    out = {}
    for ai, A in enumerate(ARCHS):
        for mi, m in enumerate(MODES):
            lw = np.array([_call(R.limit_by_warps, A, t) for t in range(1, 1101)], np.int64)
            lr = np.array([[_call(R.limit_by_registers, A, t, r, m) for r in range(301)]
                           for t in range(1, 1101)], np.int64)
            ls = np.array([R.limit_by_smem(A, s, m)
                           for s in range(A.shared_mem_per_block + 65)], np.int64)
            rwl = np.array([Rocc.register_warp_limit(A, r) for r in range(301)], np.int64)
            out[f"lw_{ai}_{mi}"] = lw
            out[f"lr_{ai}_{mi}"] = lr
            out[f"ls_{ai}_{mi}"] = ls
            out[f"rwl_{ai}_{mi}"] = rwl
    np.savez_compressed(os.path.join(HERE, "occupancy_tables.npz"), **out)


def occupancy_random(n=200_000):
    rng = random.Random(0x1701)
    rows = []
    for _ in range(n):
        ai = rng.randrange(len(ARCHS))
        A = ARCHS[ai]
        mi = rng.randrange(2)
        t = rng.randrange(0, 1101)
        r = rng.randrange(0, 301) if rng.random() < 0.9 else rng.randrange(0, 70000)
        s = rng.randrange(0, A.shared_mem_per_block + 100) if rng.random() < 0.9 \
            else rng.randrange(0, 1 << 33)
        try:
            res = R.occupancy(A, R.LaunchInput(t, r, s), MODES[mi])
            rows.append((ai, mi, t, r, s, 0, res.warps_per_block, res.limit_warps,
                         res.limit_regs, res.limit_smem, res.active_blocks, res.active_warps,
                         ("warps", "registers", "shared-memory", "illegal").index(
                             res.limiter.value),
                         np.float64(res.occupancy).view(np.int64)))
        except R.IllegalLaunchError:
            rows.append((ai, mi, t, r, s, 1, 0, 0, 0, 0, 0, 0, 3, 0))
    arr = np.array(rows, np.int64)
    np.savez_compressed(os.path.join(HERE, "occupancy_random.npz"), rows=arr)


def suggest_golden():
    rows = []
    for ai, A in enumerate(ARCHS):
        for mi, m in enumerate(MODES):
            for regs in list(range(0, 256, 3)) + [255, 256, 63, 64]:
                for smem in (0, 1, 4096, 6144, 6145, 10000, 12288, 24576, 49152, 49153,
                             232448, 232449):
                    res = R.KernelResources("k", registers_per_thread=regs,
                                            static_shared_mem=smem)
                    try:
                        s = R.suggest(A, res, m)
                        rows.append([ai, mi, regs, smem, "ok", list(s.thread_candidates),
                                     s.register_headroom, s.smem_budget,
                                     s.best_occupancy.hex(), s.best_threads, s.best_blocks])
                    except R.IllegalLaunchError:
                        rows.append([ai, mi, regs, smem, "illegal"])
    with open(os.path.join(HERE, "suggest.json"), "w") as fh:
        json.dump({"meta": META, "rows": rows}, fh)


def _ref_mix(counts_pairs, regs):
    return R.InstructionMix({R.OpClass(c.value if hasattr(c, "value") else c): n
                             for c, n in counts_pairs}, regs)


def _features(mx, cc):
    try:
        return {"cost": R.cost_estimate(mx, cc).hex(),
                "cycles": [v.hex() for v in Rmix.category_cycles(mx, cc).values()],
                "coef": [v.hex() for v in Rmix.category_coefficients(mx, cc).values()],
                "shares": [v.hex() for v in R.pipeline_utilization(mx, cc).values()],
                "per_class": {c.value: v.hex() for c, v in
                              Rmix.per_class_cycles(mx, cc).items()}}
    except R.UnsupportedArchitectureError:
        return "unsupported"


def mix_golden():
    sass = open("/root/reference/pkg/tests/data/atax_kepler.sass.txt").read()
    ((name, instrs),) = R.parse_disassembly(sass)
    mx = R.aggregate(instrs)
    atax = {"name": name, "counts": [[c.value, n] for c, n in mx.counts.items()],
            "reg_operands": mx.reg_operands, "flops": mx.flops, "mem": mx.mem,
            "ctrl": mx.ctrl, "total": mx.total_instructions,
            "intensity": R.intensity(mx).hex(),
            "instructions": [[i.opcode, list(i.modifiers), i.predicate,
                              i.register_operand_count] for i in instrs],
            "features": {str(cc): _features(mx, cc) for cc in (2.0, 3.5, 5.2, 6.0, 10.0)}}
    variants = []
    for kname in W.KERNEL_NAMES:
        for u in range(1, 6):
            for f in ("", "-use_fast_math"):
                vm = W.variant_mix(kname, u, f)
                rm = _ref_mix(list(vm.counts.items()), vm.reg_operands)
                variants.append({"kernel": kname, "unroll": u, "flag": f,
                                 "counts": [[c.value, n] for c, n in rm.counts.items()],
                                 "reg_operands": rm.reg_operands,
                                 "intensity": R.intensity(rm).hex(),
                                 "features": {str(cc): _features(rm, cc)
                                              for cc in (2.0, 3.5, 5.2, 6.0, 10.0)}})
    rng = random.Random(0xFEED)
    classes = [c for c in R.OpClass if c is not R.OpClass.REGS]
    rand = []
    for i in range(3000):
        k = rng.randrange(0, 9)
        picked = rng.sample(classes, k)
        counts = [[c.value, rng.choice((0, 1, 2, 3, 7, 13, 100, 999, 123457))
                   if rng.random() < 0.2 else rng.randrange(0, 600)] for c in picked]
        regs = rng.randrange(0, 5000)
        rm = R.InstructionMix({R.OpClass(c): n for c, n in counts}, regs)
        scale = rng.choice((1.0, 0.5, 3.0, 1e-3, 7.25))
        cc = rng.choice((2.0, 3.5, 5.2, 6.0))
        rand.append({"counts": counts, "reg_operands": regs, "scale": scale.hex(), "cc": cc,
                     "cost_scaled": R.cost_estimate(rm, cc, scale).hex(),
                     "intensity": R.intensity(rm).hex(), "features": _features(rm, cc)})
    with open(os.path.join(HERE, "mix.json"), "w") as fh:
        json.dump({"meta": META, "atax": atax, "variants": variants, "random": rand}, fh)


def _outcome_of(f):
    try:
        v = f()
    except KeyError:
        return "KeyError"
    if isinstance(v, dict):
        return {(c.value if hasattr(c, "value") else c): x.hex() for c, x in v.items()}
    return v.hex()


def partial_table_golden(n=600):
    """Partial throughput tables: each table drops a random set of
    (class, key) entries; record what cost_estimate / category_cycles /
    pipeline_utilization / per_class_cycles return or raise (KeyError)."""
    rng = random.Random(0x9A57)
    classes = [c for c in R.OpClass if c is not R.OpClass.UNCLASSIFIED]
    full = dict(Rmix.DEFAULT_THROUGHPUT.ipc)
    rows = []
    for i in range(n):
        drop = set()
        for _ in range(rng.choice((1, 1, 2, 3))):
            drop.add((rng.choice(classes), rng.choice(Rmix.SM_KEYS)))
        ipc = {k: v for k, v in full.items() if k not in drop}
        table = Rmix.ThroughputTable(ipc=ipc)
        k = rng.randrange(0, 6)
        picked = rng.sample([c for c in classes if c is not R.OpClass.REGS]
                            + [R.OpClass.UNCLASSIFIED], k)
        if rng.random() < 0.5 and drop:        # make a dropped class likely in use
            c0 = next(iter(drop))[0]
            if c0 is not R.OpClass.REGS and c0 not in picked:
                picked.append(c0)
        counts = [[c.value, rng.choice((0, 1, 5, 40))] for c in picked]
        regs = rng.choice((0, 0, 3, 77))
        mx = R.InstructionMix({R.OpClass(c): m for c, m in counts}, regs)
        cc = rng.choice((2.0, 3.5, 5.2, 6.0))
        rows.append({
            "drop": [[c.value, key] for c, key in sorted(drop, key=lambda t: (t[0].value, t[1]))],
            "counts": counts, "reg_operands": regs, "cc": cc,
            "cost": _outcome_of(lambda: R.cost_estimate(mx, cc, 1.0, table)),
            "cycles": _outcome_of(lambda: Rmix.category_cycles(mx, cc, table)),
            "shares": _outcome_of(lambda: R.pipeline_utilization(mx, cc, table)),
            "per_class": _outcome_of(lambda: Rmix.per_class_cycles(mx, cc, table))})
    with open(os.path.join(HERE, "partial_table.json"), "w") as fh:
        json.dump({"meta": META, "rows": rows}, fh)


def corpus_golden(n_kernels=2000):
    c = W.make_corpus(n_kernels)
    text = W.corpus_text(c)
    t0 = time.time()
    funcs = R.parse_disassembly(text)
    rows = []
    for name, instrs in funcs:
        mx = R.aggregate(instrs)
        rows.append([name, [[cl.value, n] for cl, n in mx.counts.items()], mx.reg_operands])
    with open(os.path.join(HERE, "corpus.json"), "w") as fh:
        json.dump({"meta": META, "n_kernels": n_kernels, "n_instr": c.n_instr,
                   "text_sha256": hashlib.sha256(text.encode()).hexdigest(),
                   "reference_seconds": time.time() - t0, "kernels": rows}, fh)


# ---------------------------------------------------------------------------
# scoring composition from reference functions (B1: separable tables)
# ---------------------------------------------------------------------------

IDX = (1 << 34) - 1


def _segment_tables(A, mode, tcs, regs, smem):
    lw = np.array([_call(R.limit_by_warps, A, t) for t in tcs], np.int64)
    lr = np.array([[_call(R.limit_by_registers, A, t, r, mode) for r in regs] for t in tcs],
                  np.int64)
    ls = np.array([R.limit_by_smem(A, s, mode) for s in smem], np.int64)
    wpb = np.array([Rocc.warps_per_block(A, t) for t in tcs], np.int64)
    return lw, lr, ls, wpb


def topk_config(cfg, mode=R.Mode.CORRECTED, verbose=True):
    """Per-segment top-k keys for a workloads.Config, via reference calls."""
    archs = [ref_arch(a) for a in cfg.archs]
    n_arch = len(archs)
    out = []
    start = 0
    for ki, kern in enumerate(cfg.kernels):
        sp = kern.space
        extras = dict(sp.extra)
        regs = extras.get("REGS", (kern.registers_per_thread,))
        smem = extras.get("SMEM", (kern.static_shared_mem,))
        rspace = R.TuningSpace(sp.thread_counts, sp.block_counts, sp.unroll_factors,
                               sp.l1_sizes_kb, sp.compiler_flags, sp.extra)
        size = R.grid_size(rspace)
        rmixes = [_ref_mix(list(m.counts.items()), m.reg_operands) for m in kern.mixes]
        for a, A in enumerate(archs):
            t0 = time.time()
            sugg = R.suggest(A, R.KernelResources("k"))
            try:
                st = set(R.static_prune(rspace, sugg).kept_thread_counts)
                lo = set(R.rule_prune(rspace, sugg, 0.0).kept_thread_counts)
                hi = set(R.rule_prune(rspace, sugg, math.inf).kept_thread_counts)
            except R.NoCandidatesError:
                st, lo, hi = set(), set(), set()
            try:
                costs = [R.cost_estimate(m, A.compute_capability) for m in rmixes]
                distinct = sorted(set(costs))
                rank_bits = [(1 << 20) - 1 - distinct.index(c) for c in costs]
            except R.UnsupportedArchitectureError:
                rank_bits = [0] * len(rmixes)
            upper = [R.intensity(m) > 4.0 for m in rmixes]
            lw, lr, ls, wpb = _segment_tables(A, mode, sp.thread_counts, regs, smem)
            nT, nB, nU, nP, nF = (len(sp.thread_counts), len(sp.block_counts),
                                  len(sp.unroll_factors), len(sp.l1_sizes_kb),
                                  len(sp.compiler_flags))
            nR, nS = len(regs), len(smem)
            best = np.zeros(0, np.uint64)
            for it, t in enumerate(sp.thread_counts):
                if lw[it] < 0:
                    continue
                # (B, U, P, F, R, S) block for this T, vectorised
                blocks = np.minimum(np.minimum(lw[it], lr[it][:, None]), ls[None, :])  # R x S
                aw = np.minimum(blocks * wpb[it], A.max_warps_per_mp)
                legal = blocks > 0
                var = (np.arange(nU)[:, None] * nF + np.arange(nF)[None, :]).reshape(-1)
                rb = np.array(rank_bits, np.uint64)[var]                      # U*F
                ru = np.array([(t in (hi if upper[v] else lo)) for v in var], np.uint64)
                stb = np.uint64(1 if t in st else 0)
                hi_bits = (np.uint64(1) << np.uint64(63)) | (ru << np.uint64(62)) | \
                    (stb << np.uint64(61)) | (rb << np.uint64(34))           # U*F
                hb = np.broadcast_to(hi_bits.reshape(1, nU, 1, nF), (nB, nU, nP, nF))
                key_hi = hb[..., None, None] | \
                    (aw.astype(np.uint64) << np.uint64(54))[None, None, None, None]
                local = (np.arange(nB * nU * nP * nF * nR * nS, dtype=np.int64)
                         .reshape(nB, nU, nP, nF, nR, nS) + it * nB * nU * nP * nF * nR * nS)
                gidx = (start + local).astype(np.uint64)
                keys = key_hi | (np.uint64(IDX) - gidx)
                keys = np.where(np.broadcast_to(legal, keys.shape), keys, np.uint64(0))
                flat = keys.reshape(-1)
                if flat.size > 64:
                    part = flat[np.argpartition(flat, flat.size - 16)[-16:]]
                else:
                    part = flat
                best = np.concatenate([best, part])
                best = np.sort(best)[::-1][:16]
            best = np.concatenate([best, np.zeros(16 - len(best), np.uint64)])
            out.append([int(x) for x in best[:cfg.k]])
            start += size
            if verbose:
                print(f"  seg k={ki} a={a}: {size} candidates, {time.time() - t0:.1f}s",
                      flush=True)
    return out


def topk_golden(name):
    cfg = W.CONFIGS[name]()
    t0 = time.time()
    res = {"meta": META, "config": cfg.name, "total": cfg.total,
           "corrected": topk_config(cfg, R.Mode.CORRECTED)}
    if name in ("config1", "config2", "config4"):
        res["verbatim"] = topk_config(cfg, R.Mode.VERBATIM)
    res["seconds"] = time.time() - t0
    with open(os.path.join(HERE, f"topk_{name}.json"), "w") as fh:
        json.dump(res, fh)


# ---------------------------------------------------------------------------
# disassembly tokenizer: reference parse_disassembly over fuzzed listings
# ---------------------------------------------------------------------------

_WS = [" ", "\t", "  ", "\xa0", "\u2003", "\x1f", "\u3000"]
_NL = ["\n", "\r\n", "\r", "\x0b", "\x0c", "\x1c", "\x85", "\u2028"]


def _rand_instr_line(rng):
    ops = list(W.corpus_opcodes()) + ["FFMA", "LDG", "BRA", "EXIT", "lower", "F2F", "X1", "Q"]
    op = rng.choice(ops)
    mods = "".join(rng.choice([".E", ".F64", ".S64", ".GE", ".AND", ".X", ".", "..", ".\u00e9", ".7"])
                   for _ in range(rng.randrange(0, 3)))
    opnds = [rng.choice(["R1", "R22", "RZ", "R٣", "R3x", "xR4", "-R5", "|R6|", "[R7+0x8]", "R8.64",
                         "[R9+R10]", "c[0x0][0x44]", "P0", "PT", "0x10", "SR_TID.X", "R²", "Rⅷ",
                         "R1\u00e9", "éR2", "R0_", " "]) for _ in range(rng.randrange(0, 5))]
    sep = rng.choice([", ", ",", " , ", ",,", ",\t"])
    body = op + mods + ((rng.choice([" ", " ", "\t", "  "]) + sep.join(opnds)) if opnds else "")
    pred = rng.choice(["", "", "", "@P0 ", "@!P1 ", "@PT ", "@!PT ", "@P ", "@Pé ", "@!P "])
    semi = rng.choice([" ;", ";", " ;", "", " ;;", "; ", " ; /* 0x0012 */"])
    addr = rng.choice(["", "/*0008*/ ", "  /* 0a8f */  ", "/*xyz*/ ", "/* 12 */"])
    ctrl = rng.choice(["", "", "[B------:R-:W-:-:S04] ", "[-:x] ", "[] "])
    wrap = rng.choice(["{}", "", "", "{", "}"])
    line = ctrl + addr + pred + body + semi
    if wrap == "{}":
        line = "{ " + line + " }"
    elif wrap:
        line = wrap + line
    tail = rng.choice(["", "", " /* 0x00 */", " /* a */ /* b */", " */", " /*", "  "])
    return rng.choice(_WS[:3]) + line + tail


def _rand_other_line(rng):
    return rng.choice([
        "Function : k" + str(rng.randrange(5)), "  Function:  k" + str(rng.randrange(5)) + "  ",
        "Function : a b", "\t.section\t.text.kern" + str(rng.randrange(3)) + ",\"ax\",@progbits",
        ".section  .text.", "L" + str(rng.randrange(3)) + ":", "  $x.y@z :  ", ".L_24:", "BB0_1 :",
        "// comment", "/* only a comment */", ".headerflags @\"EF\"", "", "   ", "{", "}",
        "9abc:", "lbl: x", "Function", "@P0", "@P0  ", "  /*0010*/  ", "\u00e9t\u00e9:",
    ])


def _rand_listing(rng):
    lines = []
    for _ in range(rng.randrange(1, 40)):
        lines.append(_rand_instr_line(rng) if rng.random() < 0.7 else _rand_other_line(rng))
    if rng.random() < 0.8:
        lines.insert(rng.randrange(0, max(1, len(lines) // 3)), rng.choice(
            ["Function : kern", "\t.section\t.text.kern,\"ax\"", "kern:"]))
    text = ""
    for ln in lines:
        text += ln + rng.choice(_NL[:1] * 6 + _NL)
    return text if rng.random() < 0.9 else text.rstrip("\n")


def _ref_summary(text):
    try:
        funcs = R.parse_disassembly(text)
    except R.StaticAnalysisError as exc:
        return ["err", type(exc).__name__, getattr(exc, "line", None), str(exc)]
    except Exception as exc:  # reference quirks (e.g. AttributeError)
        return ["err", type(exc).__name__, None, str(exc)]
    return ["ok", [[name, [[i.opcode, list(i.modifiers), i.predicate is not None,
                            i.register_operand_count] for i in instrs]] for name, instrs in funcs]]


def sass_golden(n=4000):
    rng = random.Random(0x5A55)
    cases = []
    corpus = W.corpus_text(W.make_corpus(40)).splitlines()
    for i in range(n):
        kind = i % 5
        if kind in (0, 1):
            text = _rand_listing(rng)
        elif kind == 2:                                   # mutated corpus listing
            a = rng.randrange(0, len(corpus) - 60)
            lines = corpus[a:a + rng.randrange(1, 60)]
            if rng.random() < 0.7:
                lines.insert(0, "\tFunction : k")
            for _ in range(rng.randrange(0, 4)):
                j = rng.randrange(len(lines))
                lines[j] = rng.choice([_rand_instr_line(rng), _rand_other_line(rng),
                                       lines[j].replace(";", ""), lines[j].replace(" ", "\t", 1),
                                       lines[j] + " /* 0xff */", "@!P2 " + lines[j].strip()])
            text = rng.choice(_NL[:2]).join(lines)
        elif kind == 3:                                   # acceptance-style printable fuzz
            printable = ("ABCDEFGHIJKLMNOPQRSTUVWXYZ0123456789 \t;:,.[]@/*-_'\"()\n"
                         "abcdefghijklmnopqrstuvwxyz{}!#=")
            text = "".join(rng.choice(printable) for _ in range(rng.randrange(0, 160)))
        else:                                             # latin-1 bytes / wide code points
            if rng.random() < 0.5:
                text = bytes(rng.randrange(256) for _ in range(rng.randrange(0, 120))).decode("latin-1")
            else:
                text = "".join(chr(rng.choice([rng.randrange(32, 127), rng.randrange(0x80, 0x3000),
                                               0x2028, 0x0663, 0x00b2, 0x2167, 0xd800]))
                               for _ in range(rng.randrange(0, 80)))
                text = "Function : k\n" + text
        cases.append({"text": text, "result": _ref_summary(text)})
    kinds = {}
    for c in cases:
        key = c["result"][0] if c["result"][0] == "ok" else c["result"][1]
        kinds[key] = kinds.get(key, 0) + 1
    with open(os.path.join(HERE, "sass_fuzz.json"), "w") as fh:
        json.dump({"meta": META, "outcomes": kinds, "cases": cases}, fh,
                  ensure_ascii=True)
    print("sass outcomes", kinds)


# ---------------------------------------------------------------------------
# analysis reports (occmix analyze data path, ref cli.py:105-134)
# ---------------------------------------------------------------------------

def _ref_analyze(arch, mode, res_text, sass_text, space=None, scale=1.0, dyn=0):
    """The body of cmd_analyze (ref cli.py:105-128) -> (json text | error)."""
    try:
        resources = R.parse_resource_report(res_text)
        by_name = {n: ins for n, ins in R.parse_disassembly(sass_text)}
        analyses = [R.analyze_kernel(arch, r, by_name.get(r.entry_name, []), mode,
                                     dynamic_shared_mem=dyn,
                                     space=space if space is not None else R.TuningSpace(),
                                     scale=scale)
                    for r in resources]
        text = R.to_json(R.report_dict(arch, mode, analyses))
        return {"ok": True, "sha256": hashlib.sha256(text.encode()).hexdigest(),
                "kernels": [hashlib.sha256(json.dumps(R.report.kernel_dict(a), indent=2)
                                           .encode()).hexdigest()[:16] for a in analyses],
                "text": text if len(text) < 40000 else None}
    except Exception as exc:   # noqa: BLE001
        return {"ok": False, "error": type(exc).__name__, "message": str(exc)}


REPORT_CASES = (   # (tag, arch index, mode, space spec, scale, dynamic smem)
    ("default", None, "corrected", None, 1.0, 0),
    ("verbatim", None, "verbatim", None, 1.0, 0),
    ("space_scale_dyn", None, "corrected",
     ((64, 128, 192, 256, 384, 512, 1024), (8, 16), (1, 2), (16, 48), ("", "-O3")), 2.5, 1024),
)


def report_golden(n_kernels=120):
    atax_res = open("/root/reference/pkg/tests/data/atax_kepler.ptxas.txt").read()
    atax_sass = open("/root/reference/pkg/tests/data/atax_kepler.sass.txt").read()
    c = W.make_corpus(n_kernels)
    sass = W.corpus_text(c)
    out = {"meta": META, "n_kernels": n_kernels,
           "sass_sha256": hashlib.sha256(sass.encode()).hexdigest(),
           "atax": {"ptxas": atax_res, "sass": atax_sass, "runs": []}, "corpus": []}
    for ai, A in enumerate(ARCHS):
        for tag, _, mode, sp, scale, dyn in REPORT_CASES:
            space = None if sp is None else R.TuningSpace(*sp)
            m = R.Mode(mode)
            out["atax"]["runs"].append({"arch": ai, "case": tag, "result":
                                        _ref_analyze(A, m, atax_res, atax_sass, space, scale, dyn)})
            res_text = W.corpus_resource_report(n_kernels, 1000 * ai + len(tag),
                                               A.max_regs_per_thread, A.shared_mem_per_block - dyn)
            r = _ref_analyze(A, m, res_text, sass, space, scale, dyn)
            r["text"] = None
            r["resources"] = [[x.entry_name, x.registers_per_thread, x.static_shared_mem,
                               [list(b) for b in x.const_mem_banks], x.spill_loads,
                               x.spill_stores, x.target_cc]
                              for x in R.parse_resource_report(res_text)]
            out["corpus"].append({"arch": ai, "case": tag, "seed": 1000 * ai + len(tag),
                                  "result": r})
    # error paths: registers / smem above the arch limit, scale <= 0, empty report
    errs = []
    k = R.builtin_arch("kepler")
    for tag, res_text, scale in (
            ("regs", "Compiling entry function 'kern_000001'\nptxas info : Used 300 registers\n", 1.0),
            ("smem", "Compiling entry function 'kern_000001'\nptxas info : Used 8 registers, "
                     "99999 bytes smem\n", 1.0),
            ("scale", "Compiling entry function 'kern_000001'\nptxas info : Used 8 registers\n", 0.0),
            ("empty", "ptxas info : 0 bytes gmem\n", 1.0),
            ("clause", "Compiling entry function 'k'\nptxas info : Used many registers\n", 1.0)):
        errs.append({"case": tag, "resources": res_text, "scale": scale,
                     "result": _ref_analyze(k, R.Mode.CORRECTED, res_text, sass, None, scale)})
    out["errors"] = errs
    with open(os.path.join(HERE, "report.json"), "w") as fh:
        json.dump(out, fh)
    print("report cases", sum(r["result"]["ok"] for r in out["corpus"]), "ok of",
          len(out["corpus"]))


# ---------------------------------------------------------------------------
# spec-file parsers (space files, arch INI, opcode-class tables)
# ---------------------------------------------------------------------------

def _outcome(f, text, dump):
    try:
        return ["ok", dump(f(text))]
    except R.StaticAnalysisError as exc:
        return ["err", type(exc).__name__, getattr(exc, "line", None), str(exc)]
    except Exception as exc:  # reference quirks (TypeError, raw ValueError, ...)
        return ["err", type(exc).__name__, None, str(exc)]


def _dump_space(sp):
    return [[n, list(v)] for n, v in sp._dimensions()]


def _dump_archs(specs):
    import dataclasses
    return [{k: (v.value if hasattr(v, "value") else v)
             for k, v in dataclasses.asdict(s).items()} for s in specs]


def _dump_opclasses(table):
    return [[k, v.value] for k, v in table.items()]


def _rand_space_text(rng):
    names = ["TC", "BC", "UIF", "PL", "CFLAGS", "tc", "Cflags", "X", "N_2", "uif"]
    ints = lambda: rng.choice([0, 1, 2, 5, 16, 24, 32, 48, 64, 96, 100, 192, 1025, -32, -1])

    def rhs():
        k = rng.randrange(9)
        sp = lambda: rng.choice(["", " ", "  ", "\t"])
        if k <= 2:
            args = [str(ints()) for _ in range(rng.choice([2, 2, 3, 1, 4]))]
            if rng.random() < 0.2:
                args[-1] = "0"
            return "range(" + sp() + (sp() + "," + sp()).join(args) + sp() + ")"
        if k <= 5:
            toks = []
            for _ in range(rng.randrange(0, 5)):
                toks.append(rng.choice([str(ints()), "'-use_fast_math'", "''", '"-O3"', "'",
                                        '"', "x", "1.5", " 32 ", "'a", "0x20", "+64", "- 1"]))
            return rng.choice(["[", "[ "]) + ",".join(toks) + rng.choice(["]", " ]"])
        return rng.choice(["range(1,5", "[1,2", "{1,2}", "range(a,b)", "1", "", "range(1 , 5 , 2)",
                           "[32, 64] extra", "range(-64,0,-32)"])

    if rng.random() < 0.45:                          # well-formed file
        lines = []
        for name in rng.sample(names, rng.randrange(1, 5)):
            if name.upper() == "TC":
                vals = rng.choice(["range(32,1025,32)", "[64, 128,256]", "range(64, 513, 64)",
                                   "[32]", "range(1024,0,-32)", "[96,32,96]"])
            elif name.upper() == "CFLAGS":
                vals = rng.choice(["['', '-use_fast_math']", '["-O3"]', "['a','b','c']"])
            else:
                vals = rng.choice(["range(1,6)", "[16, 48]", "range(24,193,24)", "[7]",
                                   "range( 2 , 11 , 3 )", "['x', 2]"])
            lines.append(f"param {name}[] = {vals};")
        return rng.choice(_NL[:2]).join(lines)
    lines = []
    for _ in range(rng.randrange(0, 7)):
        r = rng.random()
        if r < 0.1:
            lines.append(rng.choice(["", "   ", "# comment", "// note", "#param TC[] = [1];"]))
        elif r < 0.17:
            lines.append(rng.choice(["param TC = [32];", "parm TC[] = [32];", "param [] = [1];",
                                     "param TC[ ] = [32, 64]", "param\tBC[]\t=\t[24];;",
                                     "PARAM TC[] = [32];", "param TC[]=[32];  "]))
        else:
            lines.append(f"param {rng.choice(names)}[] = {rhs()}{rng.choice([';', ';', '', ' ;'])}")
    return rng.choice(_NL[:2]).join(lines)


def _rand_arch_text(rng):
    base = [ln for ln in W.SM100_INI.splitlines() if "=" in ln]
    sections = []
    for si in range(rng.choice([1, 1, 1, 2, 0])):
        body = list(base)
        for _ in range(rng.randrange(0, 3)):
            j = rng.randrange(len(body))
            key = body[j].split("=")[0].strip()
            op = rng.randrange(7)
            if op == 0:
                del body[j]
            elif op == 1:
                body[j] = f"{key} = {rng.choice(['abc', '1.5', '', '-4', '0', '10', '1e3', ' 7 '])}"
            elif op == 2:
                body.append(f"{rng.choice(['cuda_cores_per_mp', 'global_mem_mb', 'gpu_clock_mhz', 'mem_clock_mhz', 'constant_mem_bytes', 'l2_cache_mb', 'bogus_key'])}"
                            f" = {rng.choice(['128', '40960', 'x', '1.5', '50'])}")
            elif op == 3:
                body[j] = f"{key} = {rng.choice(['31', '33', '64', '96', '1024', '2049', '4', '255'])}"
            elif op == 4:
                body.insert(j, rng.choice(["garbage line", "; comment", "# c", "  indented = 1",
                                           "key: value", "= 3"]))
            elif op == 5:
                body[j] = "family = " + rng.choice(["KEPLER", "fermi", "volta", "other", ""])
            else:
                body.append(body[j])                               # duplicate option
        name = rng.choice(["sm100-b200", "kepler", "my arch", "x", "sm100-b200"])
        sections.append([f"[{name}]"] + body)
    lines = [ln for sec in sections for ln in sec]
    if rng.random() < 0.1:
        lines.insert(0, rng.choice(["orphan = 1", "[broken", "[]"]))
    return "\n".join(lines)


def _rand_opclass_text(rng):
    classes = [c.value for c in R.OpClass] + ["Bogus", "fp32", "Regs"]
    keys = ["FFMA", "DADD", "F2F.F64", "I2F.U32", "LDG.E.64", "IMAD", "X1", "ffma", "1ABC",
            "F2F .F64", "BRA", "MOV32I"]
    lines = []
    if rng.random() < 0.4:                           # well-formed table
        for _ in range(rng.randrange(1, 12)):
            lines.append(f"{rng.choice(keys[:8] + keys[10:])} -> "
                         f"{rng.choice([c.value for c in R.OpClass if c is not R.OpClass.REGS])}")
        return "\n".join(lines)
    for _ in range(rng.randrange(0, 8)):
        r = rng.random()
        if r < 0.1:
            lines.append(rng.choice(["", "# x", "  # y", "FFMA => FP32", "FFMA ->", "-> FP32"]))
        else:
            lines.append(f"{rng.choice(keys)}{rng.choice([' -> ', '->', '  ->\t', ' - > '])}"
                         f"{rng.choice(classes)}{rng.choice(['', '', ' ', ' extra'])}")
    return rng.choice(_NL[:2]).join(lines)


def specs_golden(n=1500):
    rng = random.Random(0x5BEC)
    out = {"meta": META, "space": [], "arch": [], "opclass": []}
    for _ in range(n):
        t = _rand_space_text(rng)
        out["space"].append({"text": t, "result": _outcome(R.parse_space_file, t, _dump_space)})
    for _ in range(n // 3):
        t = _rand_arch_text(rng)
        out["arch"].append({"text": t, "result": _outcome(R.arch.parse_arch_config, t, _dump_archs)})
    for _ in range(n // 3):
        t = _rand_opclass_text(rng)
        out["opclass"].append({"text": t, "result": _outcome(Rmix.parse_opclass_table, t,
                                                             _dump_opclasses)})
    for k in ("space", "arch", "opclass"):
        kinds = {}
        for c in out[k]:
            key = c["result"][0] if c["result"][0] == "ok" else c["result"][1]
            kinds[key] = kinds.get(key, 0) + 1
        out["outcomes_" + k] = kinds
        print(k, kinds)
    with open(os.path.join(HERE, "specs.json"), "w") as fh:
        json.dump(out, fh, ensure_ascii=True)


if __name__ == "__main__":
    steps = sys.argv[1:] or ["tables", "random", "suggest", "mix", "corpus", "config1",
                             "config2", "config4"]
    if "--big" in steps:
        steps = [s for s in steps if s != "--big"] + ["config5"]
    for s in steps:
        t0 = time.time()
        {"tables": occupancy_tables, "random": occupancy_random, "suggest": suggest_golden,
         "mix": mix_golden, "partial": partial_table_golden, "corpus": corpus_golden, "sass": sass_golden,
         "report": report_golden, "specs": specs_golden}.get(
            s, lambda: topk_golden(s))()
        print(f"{s}: {time.time() - t0:.1f}s", flush=True)
