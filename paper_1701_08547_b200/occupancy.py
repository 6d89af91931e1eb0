"""Theoretical occupancy (mirrors occmix/occupancy.py).

Value types (``Mode``, ``Limiter``, ``LaunchInput``, ``OccupancyResult``,
``SuggestionReport``; ref occupancy.py:26-82) are host-side.  Every
number is computed on the GPU: the scalar functions below are batch-of-one
calls into the Kd dump kernel (``occx_occupancy_batch``) or the K4 sweep
kernel (``occx_suggest_batch``); ``occupancy_batch`` / ``suggest_batch``
in :mod:`.batch` are the bulk entry points.  ``thread_candidates`` is an
arch-level table (ref :198-211) computed host-side once per arch when
packing membership masks.
"""

from __future__ import annotations

import enum
import functools
from dataclasses import dataclass

from .arch import ArchSpec
from .errors import IllegalLaunchError


class Mode(str, enum.Enum):
    CORRECTED = "corrected"
    VERBATIM = "verbatim"


class Limiter(str, enum.Enum):
    WARPS = "warps"
    REGISTERS = "registers"
    SHARED_MEMORY = "shared-memory"
    ILLEGAL = "illegal"


MODE_CODE = {Mode.CORRECTED: 0, Mode.VERBATIM: 1}
LIMITER_OF_CODE = (Limiter.WARPS, Limiter.REGISTERS, Limiter.SHARED_MEMORY,
                   Limiter.ILLEGAL)


@dataclass(frozen=True)
class LaunchInput:
    """(threads, registers/thread, shared bytes/block); 0 = unspecified
    (ref occupancy.py:38-52)."""

    threads_per_block: int
    regs_per_thread: int = 0
    shared_per_block: int = 0

    def __post_init__(self):
        if self.threads_per_block < 1:
            raise IllegalLaunchError("threads_per_block must be >= 1")
        if self.regs_per_thread < 0 or self.shared_per_block < 0:
            raise IllegalLaunchError("resource amounts must be non-negative")


@dataclass(frozen=True)
class OccupancyResult:
    warps_per_block: int
    limit_warps: int
    limit_regs: int
    limit_smem: int
    active_blocks: int
    active_warps: int
    occupancy: float
    limiter: Limiter
    mode: Mode


@dataclass(frozen=True)
class SuggestionReport:
    thread_candidates: tuple[int, ...]
    registers_used: int
    register_headroom: int
    smem_budget: int
    best_occupancy: float
    best_threads: int
    best_blocks: int

    @property
    def headroom_pair(self) -> tuple[int, int]:
        return (self.registers_used, self.register_headroom)


def thread_candidates(arch: ArchSpec) -> tuple[int, ...]:
    """Block sizes whose blocks tile the SM's warp budget exactly
    (ref occupancy.py:198-211).  Arch-level table, not per-candidate work:
    memoised on the four fields it reads."""
    return _thread_candidates(arch.warp_size, arch.max_warps_per_mp, arch.max_blocks_per_mp,
                              arch.max_threads_per_block)


@functools.lru_cache(maxsize=256)
def _thread_candidates(ws: int, wmp: int, bmp: int, tmax: int) -> tuple[int, ...]:
    keep = []
    for wpb in range(1, tmax // ws + 1):
        b = min(bmp, wmp // wpb)
        if b >= 1 and b * wpb == wmp:
            keep.append(wpb * ws)
    return tuple(keep)


def _one(arch, threads, regs, smem, mode):
    from .batch import occupancy_single
    return occupancy_single(arch, threads, regs, smem, mode)


def _checked(arch, threads):
    if not 1 <= threads <= arch.max_threads_per_block:
        raise IllegalLaunchError(
            f"threads_per_block {threads} outside [1, "
            f"{arch.max_threads_per_block}] for {arch.name}")


def warps_per_block(arch: ArchSpec, threads: int) -> int:
    """ceil(threads / warp_size) (ref occupancy.py:93-94); the batch kernels
    compute it per candidate, this scalar helper is plain arithmetic."""
    return -(-threads // arch.warp_size)


def limit_by_warps(arch: ArchSpec, threads: int) -> int:
    """ref occupancy.py:104-108."""
    _checked(arch, threads)
    return _one(arch, threads, 0, 0, Mode.CORRECTED).limit_warps


def register_warp_limit(arch: ArchSpec, regs_per_thread: int) -> int:
    """ref occupancy.py:111-124."""
    return _one(arch, arch.warp_size, regs_per_thread, 0, Mode.CORRECTED).reg_warp_limit


def limit_by_registers(arch: ArchSpec, threads: int, regs_per_thread: int,
                       mode: Mode = Mode.CORRECTED) -> int:
    """ref occupancy.py:127-145."""
    _checked(arch, threads)
    return _one(arch, threads, regs_per_thread, 0, mode).limit_regs


def limit_by_smem(arch: ArchSpec, shared_per_block: int,
                  mode: Mode = Mode.CORRECTED) -> int:
    """ref occupancy.py:148-160 (no thread check, like the reference)."""
    return _one(arch, arch.warp_size, 0, shared_per_block, mode).limit_smem


def occupancy(arch: ArchSpec, launch: LaunchInput,
              mode: Mode = Mode.CORRECTED) -> OccupancyResult:
    """ref occupancy.py:163-195; raises IllegalLaunchError for threads
    outside [1, max_threads_per_block] like the reference."""
    _checked(arch, launch.threads_per_block)
    r = _one(arch, launch.threads_per_block, launch.regs_per_thread,
             launch.shared_per_block, mode)
    return r.result(Mode(mode))


def suggest(arch: ArchSpec, resources, mode: Mode = Mode.CORRECTED,
            dynamic_shared_mem: int = 0) -> SuggestionReport:
    """Launch suggestion sweep (ref occupancy.py:232-279), on the GPU."""
    from .batch import suggest_batch
    return suggest_batch([(arch, resources, dynamic_shared_mem)], mode)[0]
