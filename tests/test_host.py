"""Host-side logic of the package (no GPU): architecture DB, tuning spaces
and pruning, membership masks, packing, workloads.  Mirrors the reference's
test_arch.py / test_tuning.py expectations."""

import math

import numpy as np
import pytest

from oracle import pyref
from paper_1701_08547_b200 import (ArchSpecError, NoCandidatesError, ParseError,
                                   PruneRule, TuningSpace, UnknownArchitectureError,
                                   builtin_arch, enumerate_space, grid_size, parse_space_file,
                                   resolve_arch, rule_prune, static_prune, thread_candidates)
from paper_1701_08547_b200.arch import parse_arch_config, pack_archs
from paper_1701_08547_b200.batch import (decode_key, pack_launches, pack_mixes,
                                         SignatureTable, mix_from_record)
from paper_1701_08547_b200.mix import (DEFAULT_OPCLASSES, DEFAULT_THROUGHPUT, InstructionMix,
                                       OpClass, classify_signature, cpi, parse_opclass_table,
                                       sm_key)
from paper_1701_08547_b200.occupancy import SuggestionReport
from paper_1701_08547_b200.tuning import membership_masks
from paper_1701_08547_b200 import workloads


def _sugg(arch):
    return SuggestionReport(thread_candidates(arch), 0, 0, 0, 1.0, 0, 0)


def test_builtins_and_resolution():
    k = builtin_arch("kepler")
    assert k.name == "kepler-k20" and k.max_warps_per_mp == 64
    assert resolve_arch("kepler-k20") is k and resolve_arch("KEPLER") is k
    with pytest.raises(UnknownArchitectureError):
        resolve_arch("volta")
    user = parse_arch_config(workloads.SM100_INI.replace("sm100-b200", "kepler"))
    assert resolve_arch("kepler", user).compute_capability == 10.0   # shadowing


def test_arch_invariants():
    bad = workloads.SM100_INI.replace("max_warps_per_mp = 64", "max_warps_per_mp = 63")
    with pytest.raises(ArchSpecError):
        parse_arch_config(bad)
    with pytest.raises(ParseError) as exc:
        parse_arch_config("[x]\nfoo\n")
    assert exc.value.line == 2       # same as occmix: "line 2: bad config syntax: ..."
    # occmix (arch.py:175-177) raises AttributeError on a missing section
    # header (MissingSectionHeaderError has no .errors); kept bug-compatible
    with pytest.raises(AttributeError):
        parse_arch_config("[x\nfoo")


def test_pack_archs_limits():
    a = pack_archs(workloads.all_archs())
    assert list(a["cost_key"]) == [0, 1, 2, 3, -1]
    odd = parse_arch_config(workloads.SM100_INI.replace("warp_size = 32", "warp_size = 48")
                            .replace("max_threads_per_mp = 2048", "max_threads_per_mp = 3072")
                            .replace("max_threads_per_block = 1024",
                                     "max_threads_per_block = 960"))[0]
    with pytest.raises(ArchSpecError):
        pack_archs([odd])


def test_thread_candidates_match_oracle():
    for a in workloads.all_archs():
        assert thread_candidates(a) == pyref.thread_candidates(a)


def test_grid_and_enumeration():
    assert grid_size(TuningSpace()) == 5120
    assert next(iter(enumerate_space(TuningSpace()))) == (32, 24, 1, 16, "")
    sp = parse_space_file("param TC[] = range(32,1025,32);\nparam SC[] = range(1,6);\n")
    assert grid_size(sp) == 5120 * 5
    with pytest.raises(ValueError):
        TuningSpace(thread_counts=(48,))


def test_prune_numbers():
    # test_acceptance.py:85-103 / test_tuning.py
    k = builtin_arch("kepler")
    st = static_prune(TuningSpace(), _sugg(k))
    assert (st.pruned_size, st.reduction) == (640, 0.875)
    ru = rule_prune(TuningSpace(), _sugg(k), 12.7)
    assert (ru.pruned_size, ru.reduction, ru.kept_thread_counts) == (320, 0.9375, (512, 1024))
    assert rule_prune(TuningSpace(), _sugg(k), 4.0).kept_thread_counts == (128, 256)
    f = rule_prune(TuningSpace(), _sugg(builtin_arch("fermi")), 10.0)
    assert f.kept_thread_counts == (384, 512, 768)
    assert ru.rule_applied is PruneRule.STATIC_PLUS_INTENSITY
    with pytest.raises(NoCandidatesError):
        static_prune(TuningSpace(thread_counts=(32, 64, 96)), _sugg(k))


@pytest.mark.parametrize("ai", range(5))
def test_membership_masks_match_oracle_sets(ai):
    arch = workloads.all_archs()[ai]
    for tcs in (TuningSpace().thread_counts, (32, 64, 96), (128,), tuple(range(64, 2017, 64)),
                (2048, 32, 1024, 1984)):
        sp = TuningSpace(thread_counts=tcs)
        st, lo, hi = membership_masks(sp, thread_candidates(arch))
        kept = pyref.static_kept(tcs, set(pyref.thread_candidates(arch)))
        want_lo = set(pyref.rule_kept(kept, 0.0)) if kept else set()
        want_hi = set(pyref.rule_kept(kept, math.inf)) if kept else set()
        bits = lambda m: {32 * (b + 1) for b in range(64) if (m >> b) & 1}
        assert bits(st) == set(kept) and bits(lo) == want_lo and bits(hi) == want_hi


def test_pack_launches_clamps_preserve_semantics():
    rec = pack_launches([(70000, 70000, 1 << 40), (128, 27, 0)])
    assert rec["threads"][0] == 0xFFFF and rec["regs"][0] == 0xFFFF
    assert rec["smem"][0] == 0xFFFFFFFF
    assert tuple(rec[1][["threads", "regs", "smem"]]) == (128, 27, 0)


def test_classify_and_signature_lut():
    assert classify_signature("F2F", (".F64", ".F32")) is OpClass.CONV64
    assert classify_signature("F2F", (".F32", ".F32")) is OpClass.CONV32
    assert classify_signature("FROB", ()) is OpClass.UNCLASSIFIED
    assert len(DEFAULT_OPCLASSES) == 147
    t = SignatureTable()
    assert t.intern("FFMA", ()) == 0 and t.intern("FFMA", ()) == 0
    assert t.intern("LDG", (".E",)) == 1
    assert list(t.lut()) == [0, 9]
    with pytest.raises(ParseError):
        parse_opclass_table("FADD -> Regs\n")


def test_cpi_table_bit_identical():
    m = DEFAULT_THROUGHPUT.cpi_matrix()
    for cls in OpClass:
        if cls is OpClass.UNCLASSIFIED:
            continue
        for col, cc in enumerate((2.0, 3.5, 5.2, 6.0)):
            from paper_1701_08547_b200.mix import CPI_ROW
            assert m[col, CPI_ROW[cls]] == cpi(cls, cc) == pyref.cpi(cls.value, col)
    with pytest.raises(Exception):
        sm_key(10.0)


def test_mix_packing_round_trip():
    mx = InstructionMix({OpClass.MOVE: 7, OpClass.INT_ADD32: 12, OpClass.FP32: 3}, 63)
    rec = pack_mixes([mx])[0]
    back = mix_from_record(rec)
    assert list(back.counts.items()) == list(mx.counts.items())
    assert back.reg_operands == 63


def test_decode_key():
    key = (1 << 63) | (1 << 62) | (0 << 61) | (48 << 54) | (((1 << 20) - 1 - 3) << 34) | \
        (((1 << 34) - 1) - 12345)
    d = decode_key(key)
    assert d == {"legal": True, "rule_keep": True, "static_keep": False, "active_warps": 48,
                 "rank_bits": (1 << 20) - 4, "index": 12345}


def test_workload_shapes():
    assert workloads.config1().total == 32
    assert workloads.config2().total == 26_214_400
    assert workloads.config4().total == 104_857_600
    assert workloads.config5().total == 1_284_505_600
    ints = [pyref.intensity({c.value: n for c, n in workloads.variant_mix(k, 1, "").counts.items()})
            for k in workloads.KERNEL_NAMES]
    assert [round(x, 6) for x in ints] == [3.4, 1.8, 4.6, 12.7]


def test_corpus_deterministic_and_sliceable():
    a = workloads.make_corpus(50)
    b = workloads.make_corpus(20, first=30)
    ra, rb = workloads.corpus_records(a), workloads.corpus_records(b)
    assert np.array_equal(ra[int(a.offsets[30]):], rb)
    assert (ra >> 25).max() == 0 and ((ra >> 17) & 0xFF).max() <= 4
    lengths = np.diff(a.offsets.astype(np.int64))
    assert lengths.min() >= 32 and lengths.max() <= 32 + 1984


def test_decode_matches_locate_on_random_keys():
    """ScorePlan.decode (numpy digits, zipped configs) == locate() per key,
    including weak-scaling indices beyond total and empty slots."""
    import numpy as np
    from paper_1701_08547_b200 import workloads
    from paper_1701_08547_b200.batch import IDX_MASK, ScorePlan
    cfg = workloads.config4()
    plan = object.__new__(ScorePlan)             # host-side fields only (no GPU)
    plan.kernels, plan.archs = list(cfg.kernels), list(cfg.archs)
    plan.n_arch, plan.k = len(cfg.archs), 16
    plan.n_seg = len(cfg.kernels) * plan.n_arch
    starts, dims, vb, st, nv = [], [], [], 0, 0
    for kern in cfg.kernels:
        vb.append(nv)
        nv += len(kern.mixes)
        d = [tuple(v) for _, v in kern.space._dimensions()]
        size = int(np.prod([len(x) for x in d]))
        for _ in range(plan.n_arch):
            starts.append(st)
            dims.append(d)
            st += size
    plan.seg_start, plan.seg_dims, plan.total, plan.var_base = starts, dims, st, vb
    plan.kern_dims = dims[::plan.n_arch]
    plan._seg_start_np = np.asarray(starts, np.int64)
    rng = np.random.default_rng(3)
    keys = np.zeros((plan.n_seg, plan.k), np.uint64)
    for s in range(plan.n_seg):
        n = rng.integers(0, plan.k + 1)
        size = (starts[s + 1] if s + 1 < plan.n_seg else st) - starts[s]
        idx = starts[s] + rng.integers(0, size, n) + plan.total * rng.integers(0, 3, n)
        keys[s, :n] = (np.uint64(1) << np.uint64(63)) | (np.uint64(7) << np.uint64(34)) | \
            (np.uint64(IDX_MASK) - idx.astype(np.uint64))
    for seg in plan.decode(keys):
        for e in seg.entries:
            s, cfg_t = plan.locate(e.index % plan.total)
            assert e.config == cfg_t
            ki = s // plan.n_arch
            sp = plan.kernels[ki].space
            want_v = vb[ki] + sp.unroll_factors.index(cfg_t[2]) * len(sp.compiler_flags) + \
                sp.compiler_flags.index(cfg_t[4])
            assert e.variant == want_v and e.cost_rank == (1 << 20) - 1 - 7
    assert sum(len(s.entries) for s in plan.decode(keys)) == int((keys != 0).sum())


def _py_pack(kernels, archs):
    """Python restatement of the plan blob parts (descriptors, pool, masks,
    var_kernel, mixes) for the native packer."""
    import numpy as np
    from paper_1701_08547_b200.batch import pack_mixes
    from paper_1701_08547_b200.tuning import grid_size
    pool, rows, masks, vk, mixes = [], [], [], [], []
    start = 0
    for ki, kern in enumerate(kernels):
        sp = kern.space
        ex = {n.upper(): v for n, v in sp.extra}
        dims = [sp.thread_counts, sp.block_counts, sp.unroll_factors, sp.l1_sizes_kb,
                sp.compiler_flags, ex.get("REGS", (kern.registers_per_thread,)),
                ex.get("SMEM", (kern.static_shared_mem,))]
        offs, lens = [], []
        for j, vals in enumerate(dims):
            offs.append(len(pool))
            lens.append(len(vals))
            pool += [min(int(v), 2**32 - 1) if j in (0, 1, 5, 6) else 0 for v in vals]
        size = grid_size(sp)
        for a, arch in enumerate(archs):
            rows.append((start, size, a, len(mixes), offs, lens))
            masks.append(membership_masks(sp, thread_candidates(arch)))
            start += size
        vk += [ki] * len(kern.mixes)
        mixes += list(kern.mixes)
    return rows, np.asarray(pool, np.uint32), np.asarray(masks, np.uint64).reshape(-1, 3), \
        np.asarray(vk, np.uint32), pack_mixes(mixes), start


def _native_pack(kernels, archs):
    from paper_1701_08547_b200.batch import DeviceError, _host
    from paper_1701_08547_b200.mix import DEVICE_ID
    dims = []
    for kern in kernels:
        sp = kern.space
        ex = {n.upper(): v for n, v in sp.extra}
        dims.append((sp.thread_counts, sp.block_counts, sp.unroll_factors, sp.l1_sizes_kb,
                     sp.compiler_flags, ex.get("REGS", (kern.registers_per_thread,)),
                     ex.get("SMEM", (kern.static_shared_mem,))))
    mixes = [m for k in kernels for m in k.mixes]
    return _host().pack_plan(dims, [len(k.mixes) for k in kernels], mixes,
                             [thread_candidates(a) for a in archs], DEVICE_ID, DeviceError)


def _check_native_pack(kernels, archs):
    import numpy as np
    from paper_1701_08547_b200 import _lib
    rows, pool, masks, vk, mix, total = _py_pack(kernels, archs)
    blob, offs, n_total, n_pool, starts = _native_pack(kernels, archs)
    assert n_total == total and n_pool == max(len(pool), 1)
    assert starts == [r[0] for r in rows]
    n_seg = len(rows)
    desc = np.frombuffer(blob, _lib.SEGDESC, n_seg, offs[0])
    for d, (st, size, a, vb, o, ln) in zip(desc, rows):
        assert (int(d["start"]), int(d["size"]), int(d["arch"]), int(d["var_base"])) == (st, size, a, vb)
        assert d["dim_off"].tolist() == o and d["dim_len"].tolist() == ln
    assert np.array_equal(np.frombuffer(blob, np.uint32, len(pool), offs[1]), pool)
    assert np.array_equal(np.frombuffer(blob, np.uint64, 3 * n_seg, offs[2]).reshape(-1, 3), masks)
    assert np.array_equal(np.frombuffer(blob, np.uint32, len(vk), offs[3]), vk)
    assert np.frombuffer(blob, np.uint8, mix.nbytes, offs[4]).tobytes() == mix.tobytes()


def test_native_pack_plan_matches_python_restatement():
    """csrc/occx_host.cpp pack_plan == the Python packing (membership_masks,
    value pool clamps, descriptor rows, pack_mixes) on the workloads and on
    spaces with duplicate / unsorted / numpy-int / huge thread and value
    entries."""
    import random
    import numpy as np
    from paper_1701_08547_b200 import workloads
    from paper_1701_08547_b200.batch import KernelSpec
    from paper_1701_08547_b200.mix import COUNTABLE, InstructionMix
    for cfg in (workloads.config1(), workloads.config2(), workloads.config4(), workloads.config5()):
        _check_native_pack(cfg.kernels, cfg.archs)
    rng = random.Random(5)
    archs = workloads.all_archs()
    for _ in range(60):
        kernels = []
        for kk in range(rng.randint(1, 4)):
            tc = [rng.choice(range(32, 2049, 32)) for _ in range(rng.randint(1, 14))]
            tc += rng.sample(tc, min(len(tc), rng.randint(0, 3)))          # duplicates
            if rng.random() < 0.3:
                tc = [np.int64(t) for t in tc]
            regs = tuple(rng.choice((0, 27, 255, 300, 2**40)) for _ in range(rng.randint(1, 4)))
            space = TuningSpace(tuple(tc), tuple(rng.sample(range(1, 300), rng.randint(1, 3))),
                                (1, 2)[:rng.randint(1, 2)], (16,), ("", "-use_fast_math"),
                                extra=(("REGS", regs),) if rng.random() < 0.7 else ())
            n_var = len(space.unroll_factors) * len(space.compiler_flags)
            mixes = tuple(InstructionMix({c: rng.randint(0, 2**32 - 1) for c in
                                          rng.sample(COUNTABLE, rng.randint(0, 8))},
                                         rng.randint(0, 2**62)) for _ in range(n_var))
            kernels.append(KernelSpec(f"k{kk}", space, mixes, rng.randint(0, 64),
                                      rng.randint(0, 49152)))
        _check_native_pack(kernels, rng.sample(archs, rng.randint(1, 5)))


def test_native_pack_plan_errors():
    from paper_1701_08547_b200 import workloads
    from paper_1701_08547_b200.batch import DeviceError, KernelSpec
    from paper_1701_08547_b200.mix import InstructionMix, OpClass
    arch = workloads.all_archs()[:1]
    two = (InstructionMix(), InstructionMix())
    sp = TuningSpace((64, 128), (1,), (1,), (16,), ("", "-f"), extra=(("REGS", (1, -3)),))
    with pytest.raises(ValueError, match="non-negative ints"):
        _native_pack([KernelSpec("a", sp, two)], arch)
    sp = TuningSpace((64,), (1.5,), (1,), (16,), ("", "-f"))
    with pytest.raises(ValueError, match="non-negative ints"):
        _native_pack([KernelSpec("a", sp, two)], arch)
    sp = TuningSpace((64,), (1,), (1,), (16,), ("", "-f"))
    big = (InstructionMix({OpClass.FP32: 2**32}), InstructionMix())
    with pytest.raises(DeviceError, match="above 2\\^32-1"):
        _native_pack([KernelSpec("a", sp, big)], arch)
