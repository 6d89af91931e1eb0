"""The C ABI's argument checks on a real device: every rejected call returns
the documented status (include/occx.h) and launches nothing; the Python
layer maps statuses onto the reference's exception classes."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch
    from paper_1701_08547_b200 import ScorePlan, _lib, workloads
    cfg = workloads.config1()
    plan = ScorePlan(cfg.kernels, cfg.archs, k=cfg.k)
    rec = plan.generate()
    return torch, _lib, _lib.load(), plan, rec


def test_score_topk_argument_checks(env):
    torch, L, lib, plan, rec = env
    out = torch.empty((plan.n_seg, plan.k), dtype=torch.int64, device="cuda")
    args = dict(archs=L.ptr(plan.h_archs), n_arch=plan.n_arch, rec=L.ptr(rec), n=plan.total,
                base=0, mode=0, vtab=L.ptr(plan.d_vtab), n_var=plan.n_var, n_seg=plan.n_seg,
                k=plan.k, ws=L.ptr(plan.d_ws), ws_bytes=plan.ws_bytes, out=L.ptr(out))

    def call(**kw):
        a = {**args, **kw}
        return lib.occx_score_topk(L.ctx(), a["archs"], a["n_arch"], a["rec"], a["n"], a["base"],
                                   a["mode"], a["vtab"], a["n_var"], a["n_seg"], a["k"], a["ws"],
                                   a["ws_bytes"], a["out"], L.stream_ptr())
    assert call() == 0
    assert call(k=0) == 1 and call(k=33) == 1          # OCCX_ERR_VALUE
    assert call(mode=2) == 1
    assert call(ws_bytes=8) == 1                        # workspace too small
    assert call(base=(1 << 34) - 2) == 8                # index space above 2^34: CAPACITY
    assert call(n_arch=0) != 0


def test_score_space_key_offset_capacity(env):
    torch, L, lib, plan, rec = env
    with pytest.raises(Exception):
        plan.score_implicit(0, plan.total, key_offset=(1 << 34) - plan.total + 1)
    a = plan.score_implicit(0, plan.total, key_offset=(1 << 34) - plan.total).cpu().numpy()
    b = plan.score(rec, plan.total, index_base=(1 << 34) - plan.total).cpu().numpy()
    assert np.array_equal(a, b)


def test_mix_reduce_argument_checks(env):
    torch, L, lib, plan, rec = env
    buf = torch.zeros(64, dtype=torch.uint8, device="cuda")
    off = torch.zeros(16, dtype=torch.uint8, device="cuda")
    lut = torch.zeros(4, dtype=torch.uint8, device="cuda")
    out = torch.zeros(144, dtype=torch.uint8, device="cuda")
    s = L.stream_ptr()
    assert lib.occx_mix_reduce(L.ctx(), L.ptr(buf), L.ptr(off), 1, L.ptr(lut), 0, L.ptr(out), s) == 1
    assert lib.occx_mix_reduce(L.ctx(), L.ptr(buf), L.ptr(off), 1, L.ptr(lut), 70000,
                               L.ptr(out), s) == 1
    assert lib.occx_mix_reduce(L.ctx(), L.ptr(buf) + 2, L.ptr(off), 1, L.ptr(lut), 4,
                               L.ptr(out), s) == 1      # records must be 4-byte aligned
    assert lib.occx_mix_reduce(L.ctx(), L.ptr(buf), L.ptr(off), 0, L.ptr(lut), 4, L.ptr(out), s) == 0


def test_python_layer_maps_statuses(env):
    from paper_1701_08547_b200 import (IllegalLaunchError, KernelResources,
                                       UnsupportedArchitectureError, cost_estimate,
                                       occupancy_batch, suggest_batch, workloads)
    from paper_1701_08547_b200.mix import InstructionMix, OpClass
    k20 = workloads.all_archs()[1]
    ob = occupancy_batch(k20, [(0, 0, 0), (2048, 0, 0), (128, 27, 0)])
    with pytest.raises(IllegalLaunchError):
        ob.result(0)
    with pytest.raises(IllegalLaunchError):
        ob.result(1)
    assert ob.result(2).active_blocks == 16
    with pytest.raises(IllegalLaunchError):
        suggest_batch([(k20, KernelResources("k", 300))])
    with pytest.raises(UnsupportedArchitectureError):
        cost_estimate(InstructionMix({OpClass.FP32: 3}, 0), 10.0)
    with pytest.raises(ValueError):
        cost_estimate(InstructionMix({OpClass.FP32: 3}, 0), 3.5, scale=0.0)


def test_score_space_flags_checked(env):
    torch, L, lib, plan, rec = env
    out = torch.empty((plan.n_seg, plan.k), dtype=torch.int64, device="cuda")

    def call(flags):
        return lib.occx_score_space(
            plan._ctx, L.ptr(plan.h_archs), plan.n_arch, L.ptr(plan.d_desc), plan.n_seg,
            L.ptr(plan.d_pool), plan.n_pool, 0, plan.total, 0, 0, flags, L.ptr(plan.d_vtab),
            plan.n_var, plan.n_seg, plan.k, L.ptr(plan.d_ws), plan.ws_bytes, L.ptr(out),
            L.stream_ptr())
    assert call(0) == 0 and call(L.SCORE_EVERY_KEY) == 0
    assert call(0x2) == 1                                 # unknown flag bit: ValueError


@pytest.mark.parametrize("options", [1, 2, 3, 4, 6])
def test_ctx_options_same_topk(env, options):
    """The LDG-fed K2 (two 512-thread CTAs per SM, doubled workspace) and the
    one-slice TMA ring and the dynamic tile schedules give the default's top-k
    on config 2 (golden)."""
    from helpers import load_golden
    from paper_1701_08547_b200 import ScorePlan, workloads
    torch, L, lib, _, _ = env
    h = L.ctx(options=options)
    assert lib.occx_ctx_options(h) == options
    cfg = workloads.config2()
    plan = ScorePlan(cfg.kernels, cfg.archs, k=cfg.k, options=options)
    if options & L.CTX_K2_FEED_LDG:
        assert plan.grid_lists == 2 * lib.occx_ctx_sm_count(h)
    got = plan.score(plan.generate(), plan.total).cpu().numpy().view(np.uint64)
    assert got.reshape(plan.n_seg, plan.k).tolist() == load_golden("topk_config2.json")["corrected"]


def test_k0_capacity_flags_and_64bit_register_operands(env):
    """K0 (ref mix.py:245-261, Python ints are unbounded): a kernel whose
    register operands sum past 2^32 is exact (64-bit total); a call whose
    offsets span >= 2^32 records or a kernel >= 2^29 records is flagged
    OCCX_ERR_CAPACITY per row (mix_from_record raises) instead of wrapping."""
    from paper_1701_08547_b200 import batch, _lib as L2
    from paper_1701_08547_b200.errors import DeviceError
    torch, L, lib, _, _ = env
    n = 17_000_000                                    # 255 * n > 2^32
    rec = torch.full((n,), (255 << 17) | (3 << 1), dtype=torch.int32, device="cuda")
    off = batch._to_device(np.asarray([0, n], np.uint64))
    lut = batch._to_device(batch.CLASS_LUT)
    out = batch._to_host(batch.mix_reduce(rec, off, 1, lut, len(batch.CLASS_LUT)), L2.MIX, 1)
    assert int(out[0]["reg_operands"]) == 255 * n and int(out[0]["counts"][3]) == n
    assert int(out[0]["reserved"]) == 0
    # a call spanning 2^32 records: flagged before any record is read
    off = batch._to_device(np.asarray([0, 5, 1 << 32], np.uint64))
    out = batch._to_host(batch.mix_reduce(rec, off, 2, lut, len(batch.CLASS_LUT)), L2.MIX, 2)
    assert out["reserved"].tolist() == [8, 8]
    with pytest.raises(DeviceError):
        batch.mix_from_record(out[0])
    # one kernel of 2^29 records (2 GB): flagged; its neighbour is not
    big = torch.zeros((1 << 29) + 64, dtype=torch.int32, device="cuda")
    off = batch._to_device(np.asarray([0, 64, 64 + (1 << 29)], np.uint64))
    out = batch._to_host(batch.mix_reduce(big, off, 2, lut, len(batch.CLASS_LUT)), L2.MIX, 2)
    assert out["reserved"].tolist() == [0, 8] and int(out[0]["counts"][0]) == 64
    del big


def test_workspace_scheduler_block_and_one_call_errors(env):
    """occx_score_workspace_init zeroes the scheduler block (the record
    scorer leaves it zero after every call); occx_score_space_host and
    occx_space_buf_bytes reject bad arguments before launching anything."""
    import ctypes
    from paper_1701_08547_b200.batch import _SpacePack
    torch, L, lib, plan, rec = env
    ctx = L.ctx()
    assert lib.occx_score_workspace_init(ctx, None, plan.n_seg, plan.k, L.stream_ptr()) == 1
    assert lib.occx_score_workspace_init(ctx, L.ptr(plan.d_ws), plan.n_seg, 0, L.stream_ptr()) == 1
    ws = torch.full((plan.ws_bytes,), 0x5A, dtype=torch.uint8, device="cuda")
    assert lib.occx_score_workspace_init(ctx, L.ptr(ws), plan.n_seg, plan.k, L.stream_ptr()) == 0
    lists = plan.grid_lists * plan.n_seg * plan.k * 8
    assert int(ws[lists:].sum()) == 0 and int(ws[:lists].min()) == 0x5A
    out = torch.empty((plan.n_seg, plan.k), dtype=torch.int64, device="cuda")
    for _ in range(3):                   # the block is zero again after every call
        assert lib.occx_score_topk(ctx, L.ptr(plan.h_archs), plan.n_arch, L.ptr(rec), plan.total,
                                   0, 0, L.ptr(plan.d_vtab), plan.n_var, plan.n_seg, plan.k,
                                   L.ptr(ws), plan.ws_bytes, L.ptr(out), L.stream_ptr()) == 0
        torch.cuda.synchronize()
        assert int(ws[lists:].sum()) == 0
    pk = _SpacePack(plan.kernels, plan.archs, plan.k)
    nb, off = ctypes.c_uint64(0), ctypes.c_uint64(0)
    assert lib.occx_space_buf_bytes(ctx, len(pk.blob), pk.n_var, pk.n_arch, pk.n_seg, 0,
                                    ctypes.byref(nb), ctypes.byref(off)) == 1      # k = 0
    assert lib.occx_space_buf_bytes(ctx, len(pk.blob), pk.n_var, pk.n_arch, pk.n_seg, pk.k,
                                    ctypes.byref(nb), ctypes.byref(off)) == 0
    buf = torch.empty((nb.value,), dtype=torch.uint8, device="cuda")
    blob = (ctypes.c_char * len(pk.blob)).from_buffer(pk.blob)
    keys = np.zeros((pk.n_seg, pk.k), np.uint64)
    cpi = np.zeros((4, 16))

    def call(**kw):
        a = dict(offs=(ctypes.c_uint64 * 5)(*pk.offsets), buf_bytes=nb.value, n_var=pk.n_var)
        a.update(kw)
        return lib.occx_score_space_host(ctx, L.ptr(pk.h_archs), pk.n_arch, ctypes.addressof(blob),
                                         len(pk.blob), a["offs"], pk.n_seg, pk.n_pool, a["n_var"],
                                         cpi.ctypes.data, 1.0, 0, 0, pk.total, 0, 0, 0, pk.k,
                                         L.ptr(buf), a["buf_bytes"], keys.ctypes.data,
                                         L.stream_ptr())
    assert call(buf_bytes=nb.value - 1) == 1                   # buffer too small
    assert call(offs=(ctypes.c_uint64 * 5)(1, 0, 0, 0, 0)) == 1  # misaligned part offset
    assert call(n_var=0) == 1
