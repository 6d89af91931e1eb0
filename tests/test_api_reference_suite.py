"""The reference's own unit / acceptance expectations (pkg/tests/
test_occupancy.py, test_mix.py, test_acceptance.py), run against this
package's public API.  Every number below comes from liboccx.so on the GPU
(the scalar functions are batch-of-one calls), so these are GPU tests."""

import math
import random

import pytest

from paper_1701_08547_b200 import (Category, Family, IllegalLaunchError, InstructionMix,
                                   KernelResources, LaunchInput, Limiter, Mode, OpClass,
                                   TuningSpace, UnsupportedArchitectureError, aggregate,
                                   builtin_arch, cost_estimate, grid_size, intensity,
                                   limit_by_registers, limit_by_smem, limit_by_warps, occupancy,
                                   pipeline_utilization, rule_prune, static_prune, suggest,
                                   thread_candidates)
from paper_1701_08547_b200.mix import category_coefficients, category_cycles, per_class_cycles
from paper_1701_08547_b200.occupancy import register_warp_limit, warps_per_block

pytestmark = pytest.mark.gpu

FERMI, KEPLER = builtin_arch(Family.FERMI), builtin_arch(Family.KEPLER)
MAXWELL, PASCAL = builtin_arch(Family.MAXWELL), builtin_arch(Family.PASCAL)


def res(regs=0, smem=0):
    return KernelResources("k", registers_per_thread=regs, static_shared_mem=smem)


# --- test_occupancy.py -------------------------------------------------------

def test_limit_by_warps_examples():
    assert limit_by_warps(KEPLER, 256) == 8
    assert limit_by_warps(FERMI, 192) == 8
    assert limit_by_warps(MAXWELL, 32) == 32
    assert warps_per_block(KEPLER, 33) == 2 and limit_by_warps(KEPLER, 33) == 16
    with pytest.raises(IllegalLaunchError):
        limit_by_warps(KEPLER, 0)
    with pytest.raises(IllegalLaunchError):
        limit_by_warps(KEPLER, 2048)


def test_limit_by_registers():
    assert limit_by_registers(KEPLER, 128, 27) == 16
    assert limit_by_registers(FERMI, 192, 27) == 6
    assert limit_by_registers(KEPLER, 128, 27, Mode.VERBATIM) == 0
    for arch in (FERMI, KEPLER, MAXWELL, PASCAL):
        over = arch.max_regs_per_thread + 1
        assert limit_by_registers(arch, 128, over) == 0
        assert limit_by_registers(arch, 128, over, Mode.VERBATIM) == 0
        assert limit_by_registers(arch, 128, 0) == arch.max_blocks_per_mp
    assert (register_warp_limit(KEPLER, 27), register_warp_limit(FERMI, 27),
            register_warp_limit(FERMI, 30), register_warp_limit(FERMI, 21)) == (64, 36, 34, 46)
    assert register_warp_limit(KEPLER, 0) == 64 and register_warp_limit(KEPLER, 256) == 0


def test_limit_by_smem():
    assert limit_by_smem(FERMI, 6144) == 8
    assert limit_by_smem(KEPLER, 0) == KEPLER.max_blocks_per_mp
    assert limit_by_smem(KEPLER, 50000) == 0
    assert limit_by_smem(FERMI, 6145) == 7
    assert limit_by_smem(FERMI, 6145, Mode.VERBATIM) == 8
    assert limit_by_smem(FERMI, 1) == FERMI.max_blocks_per_mp


def test_occupancy_cases():
    r = occupancy(KEPLER, LaunchInput(128, 27))
    assert (r.active_blocks, r.active_warps, r.occupancy, r.limiter) == (16, 64, 1.0, Limiter.WARPS)
    r = occupancy(FERMI, LaunchInput(192, 27))
    assert (r.active_blocks, r.active_warps, r.occupancy, r.limiter) == \
        (6, 36, 0.75, Limiter.REGISTERS)
    r = occupancy(FERMI, LaunchInput(192, 30))
    assert (r.active_blocks, r.active_warps, r.occupancy) == (5, 30, 0.625)
    r = occupancy(FERMI, LaunchInput(768, 30))
    assert (r.active_blocks, r.active_warps) == (1, 24)
    r = occupancy(FERMI, LaunchInput(192, 0, 12288))
    assert (r.limit_smem, r.limiter, r.active_blocks) == (4, Limiter.SHARED_MEMORY, 4)
    r = occupancy(KEPLER, LaunchInput(128, KEPLER.max_regs_per_thread + 1))
    assert (r.active_blocks, r.occupancy, r.limiter) == (0, 0.0, Limiter.ILLEGAL)
    assert occupancy(KEPLER, LaunchInput(128, 27, 50000)).limiter is Limiter.ILLEGAL
    with pytest.raises(IllegalLaunchError):
        occupancy(KEPLER, LaunchInput(2048))
    with pytest.raises(IllegalLaunchError):
        LaunchInput(0)
    r = occupancy(MAXWELL, LaunchInput(256, 40, 8192))
    assert r.active_blocks == min(r.limit_warps, r.limit_regs, r.limit_smem)


def test_suggest_goldens():
    s = suggest(KEPLER, res(27))
    assert (s.thread_candidates, s.headroom_pair, s.smem_budget, s.best_occupancy,
            s.best_blocks) == ((128, 256, 512, 1024), (27, 5), 3072, 1.0, 16)
    s = suggest(MAXWELL, res(30))
    assert (s.headroom_pair, s.smem_budget, s.best_occupancy) == ((30, 2), 1536, 1.0)
    s = suggest(FERMI, res(27))
    assert (s.best_occupancy, s.best_blocks, s.smem_budget) == (0.75, 6, 8192)
    s = suggest(FERMI, res(30))
    assert s.best_occupancy == pytest.approx(34 / 48) and s.headroom_pair == (30, 0)
    s = suggest(FERMI, res(21))
    assert (s.best_occupancy, s.headroom_pair, s.smem_budget, s.best_blocks) == \
        (pytest.approx(46 / 48), (21, 1), 6144, 8)
    s = suggest(FERMI, res(smem=10000))
    assert (s.best_occupancy, s.best_threads, s.best_blocks, s.smem_budget) == \
        (1.0, 384, 4, 12288)
    assert suggest(FERMI, res(smem=4096), dynamic_shared_mem=20480).best_blocks == 2
    with pytest.raises(IllegalLaunchError):
        suggest(FERMI, res(regs=64))
    with pytest.raises(IllegalLaunchError):
        suggest(FERMI, res(smem=49153))


# --- test_mix.py ----------------------------------------------------------------

class _I:
    def __init__(self, opcode, mods=(), pred=None, nreg=0):
        self.opcode, self.modifiers, self.predicate = opcode, tuple(mods), pred
        self.register_operand_count = nreg


def test_aggregate_rules():
    mx = aggregate([])
    assert mx.flops == mx.mem == mx.ctrl == mx.reg_operands == mx.total_instructions == 0
    mx = aggregate([_I("FFMA", nreg=4), _I("BRA")])
    assert (mx.flops, mx.ctrl, mx.mem, mx.reg_operands) == (1, 1, 0, 4)
    mx = aggregate([_I("LDG", nreg=2)] * 10)
    assert mx.mem == 10 and mx.reg_operands == 20
    mx = aggregate([_I("FFMA", pred="@P0", nreg=4)])
    assert mx.counts[OpClass.FP32] == 1 and mx.counts[OpClass.PREDICATE] == 1 and mx.ctrl == 1
    mx = aggregate([_I("BRA", pred="@P0")])
    assert mx.counts[OpClass.CONTROL] == 1 and OpClass.PREDICATE not in mx.counts
    # guard on an unclassified instruction still adds PredIns (SURVEY trap 4)
    mx = aggregate([_I("WEIRDOP", pred="@P0")] * 3 + [_I("FFMA")] * 3)
    assert mx.total_instructions == 9
    a = [_I("FFMA", nreg=4), _I("LDG", nreg=2)]
    b = [_I("BRA")] * 3
    assert aggregate(a + b) == aggregate(a) + aggregate(b)


FOUR = InstructionMix({OpClass.FP32: 192, OpClass.LOAD_STORE: 32, OpClass.CONTROL: 32}, 32)


def test_cost_estimate():
    assert cost_estimate(InstructionMix({}), 3.5) == 0.0
    assert cost_estimate(FOUR, 3.5) == pytest.approx(4.0)
    assert cost_estimate(FOUR.scaled(2), 3.5) == pytest.approx(2 * cost_estimate(FOUR, 3.5))
    assert cost_estimate(FOUR, 3.5, scale=3.0) == pytest.approx(3 * cost_estimate(FOUR, 3.5))
    mix = InstructionMix({OpClass.FP32: 10, OpClass.FP64: 5})
    assert cost_estimate(mix, 3.5) == pytest.approx(10 / 192 + 5 / 64)
    assert category_coefficients(mix, 3.5)[Category.FLOPS] == pytest.approx((10 / 192 + 5 / 64) / 15)
    assert category_coefficients(InstructionMix({OpClass.LOAD_STORE: 4}), 3.5)[Category.FLOPS] \
        == 1 / 192
    with pytest.raises(ValueError):
        cost_estimate(FOUR, 3.5, scale=0)
    with pytest.raises(UnsupportedArchitectureError):
        cost_estimate(FOUR, 10.0)
    m2 = InstructionMix({OpClass.FP32: 10, OpClass.FP64: 5, OpClass.LOAD_STORE: 7,
                         OpClass.MOVE: 3}, 20)
    assert per_class_cycles(m2, 3.5)[OpClass.REGS] == 20 / 32
    assert sum(category_cycles(m2, 3.5).values()) == pytest.approx(
        10 / 192 + 5 / 64 + 7 / 32 + 3 / 32 + 20 / 32)


def test_intensity_and_utilization():
    assert intensity(InstructionMix({OpClass.FP32: 127, OpClass.LOAD_STORE: 10})) == \
        pytest.approx(12.7)
    assert intensity(InstructionMix({OpClass.LOAD_STORE: 5})) == 0.0
    assert intensity(InstructionMix({})) == 0.0
    assert intensity(InstructionMix({OpClass.FP32: 1})) == math.inf
    assert all(v == 0.0 for v in pipeline_utilization(InstructionMix({}), 3.5).values())
    sh = pipeline_utilization(InstructionMix({OpClass.LOAD_STORE: 9}), 3.5)
    assert sh[Category.MEM] == 1.0 and sh[Category.FLOPS] == 0.0
    sh = pipeline_utilization(FOUR, 3.5)
    assert all(v == pytest.approx(0.25) for v in sh.values())


# --- test_acceptance.py ------------------------------------------------------------

def test_acceptance_1_to_4():
    golden = {Family.FERMI: {192, 256, 384, 512, 768}, Family.KEPLER: {128, 256, 512, 1024},
              Family.MAXWELL: {64, 128, 256, 512, 1024}, Family.PASCAL: {64, 128, 256, 512, 1024}}
    for fam, want in golden.items():
        assert set(suggest(builtin_arch(fam), res(27)).thread_candidates) == want
        assert set(thread_candidates(builtin_arch(fam))) == want
    assert suggest(KEPLER, res(27)).best_occupancy == 1.0
    assert suggest(FERMI, res(27)).best_occupancy == 0.75
    assert abs(suggest(FERMI, res(30)).best_occupancy - 0.71) <= 0.01
    for fam, regs, budget, blocks in ((Family.FERMI, 21, 6144, 8), (Family.KEPLER, 27, 3072, 16),
                                      (Family.MAXWELL, 30, 1536, 32), (Family.PASCAL, 30, 1536, 32)):
        s = suggest(builtin_arch(fam), res(regs))
        assert (s.smem_budget, s.best_blocks) == (budget, blocks)
    space = TuningSpace()
    assert grid_size(space) == 5120
    k = suggest(KEPLER, res(27))
    assert (static_prune(space, k).pruned_size, static_prune(space, k).reduction) == (640, 0.875)
    assert (rule_prune(space, k, 12.7).pruned_size, rule_prune(space, k, 12.7).reduction) == \
        (320, 0.9375)


def test_acceptance_7a_sweep_bounds():
    """Criterion 7a's 1,605,632-launch sweep through occupancy_batch."""
    import numpy as np
    from paper_1701_08547_b200.batch import occupancy_batch
    T, R, S = np.meshgrid(np.arange(32, 1025, 32), np.arange(256), np.arange(0, 49153, 1024),
                          indexing="ij")
    launches = np.stack([T.ravel(), R.ravel(), S.ravel()], 1)
    for arch in (FERMI, KEPLER, MAXWELL, PASCAL):
        ob = occupancy_batch(arch, launches)
        assert (ob.raw["status"] == 0).all()
        assert ((ob.raw["occupancy"] >= 0) & (ob.raw["occupancy"] <= 1)).all()
        assert (ob.raw["active_warps"] <= arch.max_warps_per_mp).all()


def test_acceptance_7c_linearity():
    rng = random.Random(20240501)
    classes = [c for c in OpClass if c not in (OpClass.REGS, OpClass.UNCLASSIFIED)]
    for _ in range(50):
        counts = {c: rng.randrange(0, 300) for c in rng.sample(classes, rng.randrange(1, 6))}
        mix = InstructionMix(counts, reg_operands=rng.randrange(0, 1000))
        cc = rng.choice((2.0, 3.5, 5.2, 6.0))
        k = rng.randrange(2, 8)
        assert cost_estimate(mix.scaled(k), cc) == pytest.approx(k * cost_estimate(mix, cc))
