"""Batch entry points of the B200 backend (the additions of SURVEY §8(b)).

* ``occupancy_batch``  -- Kd: OccupancyResult fields for N launches.
* ``suggest_batch``    -- K4: suggest() for many (arch, kernel) pairs.
* ``aggregate_batch``  -- K0: aggregate() for many instruction streams.
* ``feature_score``    -- K1: intensity / Eq. 6 cost / utilisation.
* ``ScorePlan`` / ``score_space`` -- K2+K3: score an Orio-style space and
  return the top-k configurations per (kernel, arch) segment.

All device memory is torch-allocated (plumbing only); every number comes
from liboccx.so.  Host code packs inputs, launches, and unpacks results.
"""

from __future__ import annotations

import bisect
import ctypes
import functools
import struct
import sys
import threading
from dataclasses import dataclass, field
from typing import NamedTuple, Sequence

import numpy as np
from itertools import chain

from . import _lib
from .arch import ArchSpec, COST_KEY_OF_MAJOR, pack_archs
from .errors import DeviceError, IllegalLaunchError
from .mix import (COUNTABLE, CPI_ROW, DEFAULT_OPCLASSES, DEFAULT_THROUGHPUT,
                  DEVICE_ID, Category, InstructionMix, OpClass, ThroughputTable,
                  classify_signature)
from .occupancy import (LIMITER_OF_CODE, MODE_CODE, Mode, OccupancyResult,
                        SuggestionReport, thread_candidates)
from .resources import register_operand_count
from .tuning import TuningSpace, grid_size, membership_masks

# CPython's float sum() changed in 3.12 (compensated); K1 follows the
# interpreter running this process.
SUM_MODE = 0 if sys.version_info >= (3, 12) else 1
U32_MAX = 0xFFFFFFFF
IDX_MASK = (1 << 34) - 1


_TORCH = None


def _torch():
    """torch, once a CUDA device is known to exist (checked on first use)."""
    global _TORCH
    if _TORCH is None:
        import torch
        if not torch.cuda.is_available():
            raise DeviceError("no CUDA device: the occx backend runs on the GPU only")
        _TORCH = torch
    return _TORCH


def _to_device(arr: np.ndarray):
    torch = _torch()
    flat = np.ascontiguousarray(arr).view(np.uint8).reshape(-1)
    t = torch.empty(max(flat.size, 1), dtype=torch.uint8, device="cuda")
    if flat.size:
        t[: flat.size].copy_(torch.from_numpy(flat))
    return t


class _DevPtr:
    """A device address inside a buffer the plan owns (passed to the C ABI)."""

    __slots__ = ("addr",)

    def __init__(self, addr: int):
        self.addr = addr

    def data_ptr(self) -> int:
        return self.addr


_HOST = None


def _host():
    """The native host module (csrc/occx_host.cpp); raises when it is not built."""
    global _HOST
    if _HOST is None:
        try:
            from . import _occx_host
        except ImportError as exc:
            raise DeviceError("paper_1701_08547_b200/_occx_host is not built; run "
                              "`python -m paper_1701_08547_b200.build`") from exc
        _HOST = _occx_host
    return _HOST


def _empty(nbytes: int):
    torch = _torch()
    return torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device="cuda")


def _to_host(t, dtype: np.dtype, count: int) -> np.ndarray:
    if count == 0:
        return np.zeros(0, dtype)
    raw = t[: count * dtype.itemsize].cpu().numpy()
    return raw.view(dtype).copy()


def _arch_list(archs) -> list[ArchSpec]:
    return [archs] if isinstance(archs, ArchSpec) else list(archs)


# ---------------------------------------------------------------------------
# Kd: occupancy dump
# ---------------------------------------------------------------------------

@dataclass
class OccBatch:
    """Columnar OccupancyResult batch (occupancy.py:55-65)."""

    raw: np.ndarray
    mode: Mode

    def __len__(self):
        return len(self.raw)

    def __getattr__(self, name):
        raw = self.__dict__.get("raw")
        if raw is not None and name in raw.dtype.names:
            return raw[name]
        raise AttributeError(name)

    @property
    def wpb(self):
        return self.raw["wpb"]

    def result(self, i: int) -> OccupancyResult:
        r = self.raw[i]
        if r["status"] == 2:
            raise IllegalLaunchError("threads_per_block outside the architecture's range")
        if r["status"]:
            raise ValueError("invalid candidate record")
        return OccupancyResult(
            warps_per_block=int(r["wpb"]), limit_warps=int(r["limit_warps"]),
            limit_regs=int(r["limit_regs"]), limit_smem=int(r["limit_smem"]),
            active_blocks=int(r["active_blocks"]), active_warps=int(r["active_warps"]),
            occupancy=float(r["occupancy"]), limiter=LIMITER_OF_CODE[int(r["limiter"])],
            mode=self.mode)


def pack_launches(launches, arch_index=None) -> np.ndarray:
    """(T, R, S) triples -> occx_cand_t records.  Values are clamped to the
    record's field widths in a way that keeps every result unchanged: any
    T > 65535, R > 65535 or S > 2^32-1 is already beyond every device-
    representable architecture's limit (arch.device_limits_ok)."""
    a = np.asarray(launches, dtype=np.int64).reshape(-1, 3)
    rec = np.zeros(len(a), _lib.CAND)
    if (a < 0).any():
        raise IllegalLaunchError("resource amounts must be non-negative")
    rec["threads"] = np.minimum(a[:, 0], 0xFFFF)
    rec["regs"] = np.minimum(a[:, 1], 0xFFFF)
    rec["smem"] = np.minimum(a[:, 2], U32_MAX)
    if arch_index is not None:
        rec["arch"] = np.asarray(arch_index, dtype=np.uint8)
    return rec


def occupancy_records(archs, d_records, n: int, mode: Mode = Mode.CORRECTED, d_out=None):
    """Device-level Kd: records already in HBM -> occx_occ_t array (device)."""
    torch = _torch()
    h_archs = _packed_archs(tuple(_arch_list(archs)))
    out = d_out if d_out is not None else _empty(n * _lib.OCC.itemsize)
    _lib.check(_lib.load().occx_occupancy_batch(
        _lib.ctx(), _lib.ptr(h_archs), len(h_archs), _lib.ptr(d_records), n,
        MODE_CODE[Mode(mode)], _lib.ptr(out), _lib.stream_ptr()), "occx_occupancy_batch")
    del torch
    return out


class _Lane(threading.local):
    """Per-thread page of pinned host memory the device reads and writes
    directly (UVA): the scalar API's one-launch path, no device buffers and
    no copies.  Allocated once per thread."""

    page = None


_LANE = _Lane()


def _lane():
    if _LANE.page is None:
        torch = _torch()
        t = torch.zeros(4096, dtype=torch.uint8, pin_memory=True)
        _LANE.page = (t, t.numpy(), t.data_ptr())
    return _LANE.page


def _sync(stream=None) -> None:
    _lib.check(_lib.load().occx_stream_sync(_lib.stream_ptr(stream)), "occx_stream_sync")


# occx_cand_t / occx_occ_t as struct layouts for the one-launch path
_REC1 = struct.Struct("<IIHHHBB")       # variant, smem, threads, blocks, regs, arch, aux
_OCC1 = struct.Struct("<8B4Id")         # wpb, lw, blocks, aw, limiter, status, -, -,
                                        # limit_regs, limit_smem, reg_warp_limit, -, occupancy


class OccRow(NamedTuple):
    """One occx_occ_t, unpacked (the scalar API's result row)."""

    warps_per_block: int
    limit_warps: int
    active_blocks: int
    active_warps: int
    limiter: int
    status: int
    limit_regs: int
    limit_smem: int
    reg_warp_limit: int
    occupancy: float

    def result(self, mode: Mode) -> OccupancyResult:
        if self.status == 2:
            raise IllegalLaunchError("threads_per_block outside the architecture's range")
        if self.status:
            raise ValueError("invalid candidate record")
        return OccupancyResult(
            warps_per_block=self.warps_per_block, limit_warps=self.limit_warps,
            limit_regs=self.limit_regs, limit_smem=self.limit_smem,
            active_blocks=self.active_blocks, active_warps=self.active_warps,
            occupancy=self.occupancy, limiter=LIMITER_OF_CODE[self.limiter], mode=mode)


def occupancy_single(arch, threads: int, regs: int, smem: int,
                     mode: Mode = Mode.CORRECTED) -> OccRow:
    """occupancy() of one launch: the record and the result live in pinned
    host memory the kernel reads and writes over UVA -- one launch and one
    stream synchronize (ref occupancy.py:163-195).  Same clamps as
    pack_launches."""
    if threads < 0 or regs < 0 or smem < 0:
        raise IllegalLaunchError("resource amounts must be non-negative")
    _, page, base = _lane()
    _REC1.pack_into(page, 0, 0, min(smem, U32_MAX), min(threads, 0xFFFF), 0,
                    min(regs, 0xFFFF), 0, 0)
    h_archs = _packed_archs((arch,))
    _lib.check(_lib.load().occx_occupancy_batch(
        _lib.ctx(), h_archs.ctypes.data, 1, base, 1, MODE_CODE[Mode(mode)], base + 256,
        _lib.stream_ptr()), "occx_occupancy_batch")
    _sync()
    v = _OCC1.unpack_from(page, 256)
    return OccRow(v[0], v[1], v[2], v[3], v[4], v[5], v[8], v[9], v[10], v[12])


def occupancy_batch(archs, launches, mode: Mode = Mode.CORRECTED, arch_index=None) -> OccBatch:
    """occupancy() for many launches on the GPU (ref occupancy.py:163-195)."""
    mode = Mode(mode)
    rec = pack_launches(launches, arch_index)
    d_rec = _to_device(rec)
    out = occupancy_records(archs, d_rec, len(rec), mode)
    return OccBatch(_to_host(out, _lib.OCC, len(rec)), mode)


# ---------------------------------------------------------------------------
# K4: suggest
# ---------------------------------------------------------------------------

def suggest_batch(requests, mode: Mode = Mode.CORRECTED,
                  raise_first: bool = True) -> list[SuggestionReport]:
    """suggest(arch, resources, mode, dynamic_shared_mem) for many requests
    (ref occupancy.py:232-279).  requests: (arch, resources[, dynamic]).
    With ``raise_first=False`` a failing request yields the exception the
    reference would raise, in place, instead of raising it."""
    mode = Mode(mode)
    archs: list[ArchSpec] = []
    index: dict[int, int] = {}
    inp = np.zeros(len(requests), _lib.SUGG_IN)
    for i, req in enumerate(requests):
        arch, res = req[0], req[1]
        dyn = req[2] if len(req) > 2 else 0
        if id(arch) not in index:
            index[id(arch)] = len(archs)
            archs.append(arch)
        regs = res.registers_per_thread
        smem = res.static_shared_mem + dyn
        if regs < 0 or smem < 0:
            raise ValueError("negative resource footprint")
        inp[i] = (index[id(arch)], min(regs, U32_MAX), min(smem, U32_MAX), 0)
    if not requests:
        return []
    h_archs = _packed_archs(tuple(archs))
    if len(inp) == 1:                  # the scalar API: one launch on the lane page
        _, page, base = _lane()
        page[:inp.nbytes] = inp.view(np.uint8)
        d_in, d_out = _DevPtr(base), _DevPtr(base + 256)
    else:
        d_in = _to_device(inp)
        d_out = _empty(len(inp) * _lib.SUGG.itemsize)
    _lib.check(_lib.load().occx_suggest_batch(
        _lib.ctx(), _lib.ptr(h_archs), len(h_archs), _lib.ptr(d_in), len(inp),
        MODE_CODE[mode], _lib.ptr(d_out), _lib.stream_ptr()), "occx_suggest_batch")
    if len(inp) == 1:
        _sync()
        out = page[256:256 + _lib.SUGG.itemsize].view(_lib.SUGG).copy()
    else:
        out = _to_host(d_out, _lib.SUGG, len(inp))
    reports = []
    for i, req in enumerate(requests):
        arch, res = req[0], req[1]
        o = out[i]
        st = int(o["status"])
        err = None
        if st == 2:
            regs, smem = res.registers_per_thread, int(inp[i]["smem"])
            if regs > arch.max_regs_per_thread:          # occupancy.py:245-248
                err = IllegalLaunchError(
                    f"{regs} registers/thread exceeds the {arch.max_regs_per_thread} "
                    f"supported by {arch.name}")
            else:                                        # occupancy.py:249-252
                err = IllegalLaunchError(
                    f"{smem} bytes of shared memory exceeds the "
                    f"{arch.shared_mem_per_block}-byte block capacity of {arch.name}")
        elif st == 10:
            err = IndexError("tuple index out of range")
        elif st:
            try:
                _lib.check(st, "occx_suggest_batch")
            except Exception as exc:   # noqa: BLE001 -- mapped status
                err = exc
        if err is not None:
            if raise_first:
                raise err
            reports.append(err)
            continue
        reports.append(SuggestionReport(
            thread_candidates=thread_candidates(arch),
            registers_used=res.registers_per_thread,
            register_headroom=int(o["register_headroom"]),
            smem_budget=int(o["smem_budget"]),
            best_occupancy=float(o["best_occupancy"]),
            best_threads=int(o["best_threads"]),
            best_blocks=int(o["best_blocks"])))
    return reports


# ---------------------------------------------------------------------------
# K0: aggregate
# ---------------------------------------------------------------------------

# Identity class table: K0 over "class records" (the record's 16-bit id field
# holds classify() of its signature, computed once per distinct signature on
# the host).  A 15-entry table keeps every K0 class lookup conflict-free.
CLASS_LUT = np.arange(15, dtype=np.uint8)


def classify_records(records: np.ndarray, sig_class: np.ndarray) -> np.ndarray:
    """Signature-id records -> class records (id field = sig_class[id])."""
    r = np.asarray(records, np.uint32)
    cls = np.asarray(sig_class, np.uint32)[(r >> np.uint32(1)) & np.uint32(0xFFFF)]
    return (r & np.uint32(0xFFFE0001)) | (cls << np.uint32(1))


class SignatureTable:
    """Interns (opcode, modifiers) signatures; the LUT holds classify()
    of each signature (ref mix.py:176-187), evaluated once per distinct
    signature rather than once per instruction."""

    def __init__(self, table: dict[str, OpClass] = DEFAULT_OPCLASSES):
        self.table = table
        self.ids: dict[tuple, int] = {}
        self.classes: list[int] = []

    def intern(self, opcode: str, modifiers) -> int:
        key = (opcode, tuple(modifiers))
        sid = self.ids.get(key)
        if sid is None:
            sid = len(self.classes)
            if sid >= 65535:
                raise DeviceError("more than 65535 distinct instruction signatures")
            self.ids[key] = sid
            self.classes.append(DEVICE_ID[classify_signature(opcode, key[1], self.table)])
        return sid

    def lut(self) -> np.ndarray:
        return np.asarray(self.classes or [DEVICE_ID[OpClass.UNCLASSIFIED]], np.uint8)


def pack_instructions(kernels, sigs: SignatureTable):
    """Instruction streams -> (u32 class records, u64 CSR offsets): the id
    field holds classify() of the instruction's signature (interned, so
    classify() runs once per distinct signature); reduce with CLASS_LUT."""
    recs: list[int] = []
    offs = [0]
    classes = sigs.classes
    for instrs in kernels:
        for ins in instrs:
            sid = classes[sigs.intern(ins.opcode, ins.modifiers)]
            nreg = register_operand_count(ins)
            if nreg > 255:
                raise DeviceError("instruction with more than 255 register operands")
            recs.append((1 if ins.predicate else 0) | (sid << 1) | (nreg << 17))   # OCCX_INSTR
        offs.append(len(recs))
    return np.asarray(recs, np.uint32), np.asarray(offs, np.uint64)


def mix_reduce(d_instr, d_off, n_kernels: int, d_lut, n_sig: int, d_out=None):
    """Device-level K0: CSR records in HBM -> occx_mix_t array (device)."""
    out = d_out if d_out is not None else _empty(n_kernels * _lib.MIX.itemsize)
    _lib.check(_lib.load().occx_mix_reduce(
        _lib.ctx(), _lib.ptr(d_instr), _lib.ptr(d_off), n_kernels, _lib.ptr(d_lut), n_sig,
        _lib.ptr(out), _lib.stream_ptr()), "occx_mix_reduce")
    return out


def mix_from_record(m) -> InstructionMix:
    """occx_mix_t -> InstructionMix with dict insertion order restored."""
    if int(m["reserved"]):
        raise DeviceError("instruction stream too long for the mix reducer "
                          "(>= 2^29 instructions in a kernel or 2^32 in a call)")
    present = [(int(m["first_key"][c]), c) for c in range(15) if m["counts"][c]]
    present.sort()
    counts = {COUNTABLE[c]: int(m["counts"][c]) for _, c in present}
    return InstructionMix(counts, int(m["reg_operands"]))


def aggregate_batch(kernels, table: dict[str, OpClass] = DEFAULT_OPCLASSES) -> list[InstructionMix]:
    """aggregate() over many instruction streams on the GPU (K0)."""
    kernels = [list(k) for k in kernels]
    if not kernels:
        return []
    sigs = SignatureTable(table)
    rec, off = pack_instructions(kernels, sigs)
    d_out = mix_reduce(_to_device(rec), _to_device(off), len(kernels), _to_device(CLASS_LUT),
                       len(CLASS_LUT))
    out = _to_host(d_out, _lib.MIX, len(kernels))
    return [mix_from_record(m) for m in out]


# ---------------------------------------------------------------------------
# K1: feature scoring
# ---------------------------------------------------------------------------

_CATS = (Category.FLOPS, Category.MEM, Category.CTRL, Category.REG)
_CPI_CLASS = {row: cls for cls, row in CPI_ROW.items()}


def pack_mixes(mixes: Sequence[InstructionMix]) -> np.ndarray:
    """InstructionMix objects -> occx_mix_t rows; first_key = insertion rank."""
    n = len(mixes)
    # flat (row*16 + device id, count, insertion rank) columns (C-level
    # iteration over the dicts), one numpy scatter
    dicts = [m.counts for m in mixes]
    lens = np.fromiter(map(len, dicts), np.int64, n)
    ids = np.fromiter(map(DEVICE_ID.__getitem__, chain.from_iterable(dicts)), np.int64)
    vals = list(chain.from_iterable(d.values() for d in dicts))
    regs = [m.reg_operands for m in mixes]
    starts = np.cumsum(lens) - lens
    rows = np.repeat(np.arange(n, dtype=np.int64), lens)
    ranks = np.arange(len(ids), dtype=np.int64) - np.repeat(starts, lens)
    cell = 16 * rows + ids
    # occx_mix_t as 36 u32 words: counts[16] | first_key[16] | reg_operands
    # (u64 lo, hi) | n_instr | reserved
    words = np.zeros((n, 36), np.uint32)
    words[:, 16:32] = U32_MAX
    flat = words.reshape(-1)
    if vals:
        if max(vals) > U32_MAX:
            raise DeviceError("per-class count above 2^32-1")
        cell += 20 * rows                           # row*16+d -> row*36+d
        flat[cell] = vals
        flat[cell + 16] = ranks
    r = np.asarray(regs, np.uint64)
    words[:, 32] = r & np.uint64(U32_MAX)
    words[:, 33] = r >> np.uint64(32)
    words[:, 34] = np.minimum(words[:, :16].sum(axis=1, dtype=np.uint64), U32_MAX)
    return words.view(_lib.MIX).reshape(n)


def _nonneg_ints(vals) -> np.ndarray:
    """A space dimension's values as int64 (clamped to 2^32-1); they must be
    non-negative Python/numpy ints."""
    arr = np.asarray(vals)
    if arr.dtype.kind not in "iu" or arr.ndim != 1:
        if any((not isinstance(v, int)) or v < 0 for v in vals):
            raise ValueError("TC/BC/REGS/SMEM values must be non-negative ints")
        return np.asarray([min(int(v), U32_MAX) for v in vals], np.int64)
    if arr.size and arr.min() < 0:
        raise ValueError("TC/BC/REGS/SMEM values must be non-negative ints")
    return arr.astype(np.int64)


def cost_key_of_cc(cc: float) -> int:
    return COST_KEY_OF_MAJOR.get(int(cc), -1)


@dataclass
class Features:
    cost: float
    coefficients: dict
    cycles: dict
    shares: dict
    per_class_map: dict | None      # None: a class in use has no CPI entry

    @property
    def per_class(self) -> dict:
        """per_class_cycles (ref mix.py:309-318): raises KeyError like the
        reference when the table lacks a row the mix uses, independently of
        whether the cost lookups succeeded."""
        if self.per_class_map is None:
            raise KeyError("throughput table has no entry for a class in use")
        return self.per_class_map


@dataclass
class FeatureBatch:
    sums: np.ndarray      # occx_mixsum_t[n_mix]
    feat: np.ndarray      # occx_feat_t[n_mix * n_col]
    n_col: int
    mixes: list = field(default_factory=list)
    ccs: list = field(default_factory=list)

    @property
    def intensity(self) -> list[float]:
        return [float(x) for x in self.sums["intensity"]]

    def one(self, m: int, j: int, need_cost: bool = True) -> Features:
        # one C-level conversion of the row: (cost, coef, cycles, shares,
        # per_class, status, pc_status)
        cost, coef, cyc, shares, pcl, st, pc_st = self.feat[m * self.n_col + j].tolist()
        cc = self.ccs[j]
        if st == 3:
            from .mix import sm_key
            sm_key(cc)                      # raises UnsupportedArchitectureError
        if st == 9 and need_cost:
            raise KeyError("throughput table has no entry for a class in use")
        if st not in (0, 9):
            _lib.check(st, "occx_feature_score")
        mix = self.mixes[m]
        per_class = None
        if pc_st == 0:
            per_class = {}
            for cls, n in mix.counts.items():
                if cls is not OpClass.UNCLASSIFIED and n:
                    per_class[cls] = pcl[CPI_ROW[cls]]
            if mix.reg_operands:
                per_class[OpClass.REGS] = pcl[CPI_ROW[OpClass.REGS]]
        return Features(cost=cost, coefficients=dict(zip(_CATS, coef)),
                        cycles=dict(zip(_CATS, cyc)), shares=dict(zip(_CATS, shares)),
                        per_class_map=per_class)


def feature_records(d_mix, n_mix: int, cols: Sequence[int], cpi: np.ndarray, scale: float,
                    sum_mode: int = SUM_MODE, d_sum=None, d_feat=None):
    """Device-level K1 -> (d_sum, d_feat) (allocated unless given)."""
    h_cols = np.asarray(list(cols) or [0], np.int32)
    h_cpi = np.ascontiguousarray(cpi, np.float64).reshape(4, 16)
    if d_sum is None:
        d_sum = _empty(n_mix * _lib.MIXSUM.itemsize)
    if d_feat is None:
        d_feat = _empty(n_mix * max(len(cols), 1) * _lib.FEAT.itemsize)
    _lib.check(_lib.load().occx_feature_score(
        _lib.ctx(), _lib.ptr(d_mix), n_mix, _lib.ptr(h_cols), len(cols), _lib.ptr(h_cpi),
        float(scale), sum_mode, _lib.ptr(d_sum), _lib.ptr(d_feat) if cols else None,
        _lib.stream_ptr()), "occx_feature_score")
    return d_sum, d_feat


_MIX1 = struct.Struct("<32IQII")        # occx_mix_t: counts[16] first_key[16] regs n_instr rsv


def _pack_mix_into(page, mix) -> None:
    """One InstructionMix as occx_mix_t at the start of `page` (pack_mixes
    for a single mix, without numpy)."""
    w = [0] * 16 + [U32_MAX] * 16
    total = 0
    for rank, (cls, c) in enumerate(mix.counts.items()):
        if c > U32_MAX:
            raise DeviceError("per-class count above 2^32-1")
        d = DEVICE_ID[cls]
        w[d] = c
        w[16 + d] = rank
        total += c
    if mix.reg_operands >= 1 << 64:
        raise DeviceError("reg_operands above 2^64-1")
    _MIX1.pack_into(page, 0, *w, mix.reg_operands, min(total, U32_MAX), 0)


def feature_score(mixes, ccs, scale: float = 1.0,
                  table: ThroughputTable = DEFAULT_THROUGHPUT,
                  sum_mode: int = SUM_MODE) -> FeatureBatch:
    """K1 over mixes x compute capabilities (ref mix.py:268-352)."""
    mixes = list(mixes)
    ccs = list(ccs)
    cols = [cost_key_of_cc(cc) for cc in ccs]
    if len(mixes) == 1 and len(cols) <= 1:       # the scalar API: one launch on the lane page
        _, page, base = _lane()
        _pack_mix_into(page, mixes[0])
        feature_records(_DevPtr(base), 1, cols, table.cpi_matrix(), scale, sum_mode,
                        d_sum=_DevPtr(base + 256), d_feat=_DevPtr(base + 512))
        _sync()
        sums = page[256:256 + _lib.MIXSUM.itemsize].view(_lib.MIXSUM).copy()
        feat = (page[512:512 + _lib.FEAT.itemsize].view(_lib.FEAT).copy() if cols
                else np.zeros(0, _lib.FEAT))
        return FeatureBatch(sums, feat, len(cols), mixes, ccs)
    pm = pack_mixes(mixes)
    d_sum, d_feat = feature_records(_to_device(pm), len(mixes), cols, table.cpi_matrix(),
                                    scale, sum_mode)
    sums = _to_host(d_sum, _lib.MIXSUM, len(mixes))
    feat = _to_host(d_feat, _lib.FEAT, len(mixes) * len(cols)) if cols else np.zeros(0, _lib.FEAT)
    return FeatureBatch(sums, feat, len(cols), mixes, ccs)


# ---------------------------------------------------------------------------
# K2 + K3: search-space scoring
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class KernelSpec:
    """One kernel of a search: its tuning space and one InstructionMix per
    (unroll factor, compiler flag) variant, UIF-major.  Registers / shared
    memory per candidate come from the space's extra dimensions named
    ``REGS`` / ``SMEM`` when present, else from these defaults."""

    name: str
    space: TuningSpace
    mixes: tuple
    registers_per_thread: int = 0
    static_shared_mem: int = 0

    def n_variants(self) -> int:
        return len(self.space.unroll_factors) * len(self.space.compiler_flags)


def _ranked_type():
    try:
        from ._occx_host import Ranked as R
    except ImportError:          # the module is required on use (_host()); keep import cheap
        return None
    return R


# One entry of a segment's top-k list, decoded from its key: a C struct
# sequence (index, config, variant, arch, active_warps, rule_keep,
# static_keep, cost_rank, key), built by the native decoder.
Ranked = _ranked_type()


@dataclass
class SegmentTopK:
    kernel: str
    arch: str
    entries: list


def decode_key(key: int) -> dict:
    key = int(key)
    rb = (key >> 34) & 0xFFFFF
    return {"legal": bool(key >> 63), "rule_keep": bool((key >> 62) & 1),
            "static_keep": bool((key >> 61) & 1), "active_warps": (key >> 54) & 0x7F,
            "rank_bits": rb, "index": IDX_MASK - (key & IDX_MASK)}


@functools.lru_cache(maxsize=64)
def _packed_archs(archs: tuple) -> np.ndarray:
    """occx_arch_t rows of an arch tuple: an arch-level table (like
    thread_candidates), memoised on the frozen specs."""
    out = pack_archs(archs)
    out.setflags(write=False)
    return out


class _SpacePack:
    """The host side of a (kernels x archs) search: the packed space
    description (csrc/occx_host.cpp pack_plan: segment descriptors, value
    pool, membership masks, variant -> kernel, mixes; one H2D blob) and what
    decoding keys needs.  Segment s = kernel * n_arch + arch."""

    def __init__(self, kernels, archs, k: int):
        if not 1 <= k <= 32:
            raise ValueError("k must be in [1, 32]")
        self.kernels = list(kernels)
        self.archs = list(archs)
        self.k = k
        self.n_arch = len(self.archs)
        self.n_seg = len(self.kernels) * self.n_arch
        self.h_archs = _packed_archs(tuple(self.archs))
        mixes, self.var_base, var_counts = [], [], []
        dims_all, self.kern_dims = [], []
        for kern in self.kernels:
            n_v = len(kern.mixes)
            if n_v != kern.n_variants():
                raise ValueError(f"{kern.name}: need one mix per (UIF, CFLAGS) variant")
            self.var_base.append(len(mixes))
            var_counts.append(n_v)
            mixes += kern.mixes
            sp = kern.space
            regs, smem = (kern.registers_per_thread,), (kern.static_shared_mem,)
            if sp.extra:
                names = [n.upper() for n, _ in sp.extra]
                if any(n not in ("REGS", "SMEM") for n in names) or names not in (
                        ["REGS"], ["SMEM"], ["REGS", "SMEM"]):
                    raise ValueError("extra dimensions must be REGS and/or SMEM, in that order")
                extras = {name.upper(): vals for name, vals in sp.extra}
                regs, smem = extras.get("REGS", regs), extras.get("SMEM", smem)
            dims_all.append((sp.thread_counts, sp.block_counts, sp.unroll_factors,
                             sp.l1_sizes_kb, sp.compiler_flags, regs, smem))
            self.kern_dims.append([tuple(v) for _, v in sp._dimensions()])
        self.mixes = mixes
        self.n_var = len(mixes)
        self.var_counts = var_counts
        (self.blob, self.offsets, self.total, self.n_pool,
         self.seg_start) = _host().pack_plan(dims_all, var_counts, mixes,
                                             [thread_candidates(a) for a in self.archs],
                                             DEVICE_ID, DeviceError)
        if self.total > IDX_MASK + 1:
            raise DeviceError("search space above 2^34 candidates")

    @property
    def seg_dims(self) -> list:
        return [d for d in self.kern_dims for _ in range(self.n_arch)]

    def decode(self, keys) -> list[SegmentTopK]:
        """[n_seg, k] keys -> per-segment Ranked entries (native: key fields,
        global index -> enumerate_space digits, last dimension fastest, ref
        tuning.py:70-77).  Indices of weak-scaling copies are taken modulo
        total."""
        keys = np.asarray(keys.cpu().numpy() if hasattr(keys, "cpu") else keys)
        keys = np.ascontiguousarray(keys).view(np.uint64).reshape(self.n_seg, self.k)
        segs = _host().decode(keys, self.n_arch, self.k, self.total, self.seg_start,
                              self.kern_dims, self.var_base)
        names = [a.name for a in self.archs]
        na = self.n_arch
        return [SegmentTopK(self.kernels[s // na].name, names[s % na], e)
                for s, e in enumerate(segs)]


class ScorePlan:
    """Device-resident tables for scoring a fixed (kernels x archs) search.

    Construction runs K1 (features of every variant on every arch) and the
    feature-table kernel on the GPU; host work is limited to packing the
    arch rows, the T* membership masks (tuning.membership_masks) and the
    Cartesian segment descriptors.  Segment s = kernel * n_arch + arch.
    """

    def __init__(self, kernels: Sequence[KernelSpec], archs: Sequence[ArchSpec],
                 mode: Mode = Mode.CORRECTED, k: int = 16,
                 table: ThroughputTable = DEFAULT_THROUGHPUT, scale: float = 1.0,
                 options: int = 0):
        """``options``: occx context options (_lib.CTX_*), implementation
        choices of the record scorer with identical results."""
        if not 1 <= k <= 32:
            raise ValueError("k must be in [1, 32]")
        self._ctx = _lib.ctx(options=options)
        pk = _SpacePack(kernels, archs, k)
        self._pack = pk
        self.kernels, self.archs, self.k = pk.kernels, pk.archs, k
        self.mode = Mode(mode)
        self.n_arch, self.n_seg, self.n_var = pk.n_arch, pk.n_seg, pk.n_var
        self.h_archs = pk.h_archs
        self.var_base, self.kern_dims, self.seg_start = pk.var_base, pk.kern_dims, pk.seg_start
        self.total, self.n_pool, self.mixes = pk.total, pk.n_pool, pk.mixes
        self.seg_dims = pk.seg_dims
        blob, offsets = pk.blob, pk.offsets
        var_kernel = [ki for ki, nv in enumerate(pk.var_counts) for _ in range(nv)]
        self.var_kernel = np.asarray(var_kernel, np.uint32)
        self._seg_start_np = np.asarray(self.seg_start, np.int64)
        self._blob, self._offsets = blob, offsets
        # bytes this plan copied host -> device (the space description; the
        # arch rows and CPI table travel in the kernel parameter blocks)
        self.h2d_bytes = int(len(blob) + self.h_archs.nbytes + 4 * 16 * 8)
        # one device buffer: the space description (H2D) | K1 sums | K1
        # features | feature table | K2 workspace
        ws = ctypes_u64()
        _lib.check(_lib.load().occx_score_workspace_bytes(self._ctx, self.n_seg, k,
                                                          ws.ref()), "workspace")
        self.ws_bytes = ws.value
        # per-CTA partial tables K2 leaves in the workspace (score_partials)
        self.grid_lists = _lib.load().occx_score_lists(self._ctx)
        n_cell = self.n_var * self.n_arch
        parts = [len(blob), self.n_var * _lib.MIXSUM.itemsize, n_cell * _lib.FEAT.itemsize,
                 n_cell * _lib.VENT.itemsize, self.ws_bytes]
        offs, total_b = [], 0
        for nb in parts:
            offs.append(total_b)
            total_b += -(-max(nb, 1) // 256) * 256
        self._d_buf = _empty(total_b)
        self._d_buf[:len(blob)].copy_(_torch().frombuffer(blob, dtype=_torch().uint8))
        base = self._d_buf.data_ptr()
        self.d_desc, self.d_pool, self.d_masks, self.d_var_kernel, d_mix = (
            _DevPtr(base + o) for o in offsets)
        self.d_sum, self.d_feat, self.d_vtab, self.d_ws = (_DevPtr(base + o) for o in offs[1:])
        # the workspace's scheduler block starts zeroed (the scorer leaves it zero)
        _lib.check(_lib.load().occx_score_workspace_init(
            self._ctx, _lib.ptr(self.d_ws), self.n_seg, k, _lib.stream_ptr()),
            "occx_score_workspace_init")
        # K1 on device, then the feature table
        cols = [int(a["cost_key"]) for a in self.h_archs]
        feature_records(d_mix, self.n_var, cols, table.cpi_matrix(), scale,
                        d_sum=self.d_sum, d_feat=self.d_feat)
        _lib.check(_lib.load().occx_build_vtab(
            _lib.ctx(), _lib.ptr(self.d_sum), _lib.ptr(self.d_feat), self.n_var, self.n_arch,
            _lib.ptr(self.d_var_kernel), _lib.ptr(self.d_masks),
            _lib.ptr(self.d_vtab), _lib.stream_ptr()), "occx_build_vtab")

    @property
    def masks(self) -> np.ndarray:
        """[n_seg, 3] u64 (static, rule-lower, rule-upper) membership masks."""
        o = self._offsets[2]
        return np.frombuffer(self._blob, np.uint64, 3 * self.n_seg, o).reshape(self.n_seg, 3)

    # -- candidates ---------------------------------------------------------
    def generate(self, begin: int = 0, n: int | None = None, out=None):
        """Candidates [begin, begin+n) as occx_cand_t records in HBM."""
        n = self.total - begin if n is None else n
        out = out if out is not None else _empty(n * 16)
        _lib.check(_lib.load().occx_gen_space(
            self._ctx, _lib.ptr(self.d_desc), self.n_seg, _lib.ptr(self.d_pool), begin, n,
            _lib.ptr(out), _lib.stream_ptr()), "occx_gen_space")
        return out

    def records_host(self, begin: int = 0, n: int | None = None) -> np.ndarray:
        n = self.total - begin if n is None else n
        return _to_host(self.generate(begin, n), _lib.CAND, n)

    # -- scoring ------------------------------------------------------------
    def score(self, d_records, n: int, index_base: int = 0, out=None, stream=None):
        """K2+K3 over n records in HBM -> device u64 [n_seg, k] top-k keys."""
        torch = _torch()
        # K3 writes every entry of the [n_seg, k] table: no zero-fill needed
        out = out if out is not None else torch.empty((self.n_seg, self.k), dtype=torch.int64,
                                                      device="cuda")
        _lib.check(_lib.load().occx_score_topk(
            self._ctx, _lib.ptr(self.h_archs), self.n_arch, _lib.ptr(d_records), n, index_base,
            MODE_CODE[self.mode], _lib.ptr(self.d_vtab), self.n_var, self.n_seg, self.k,
            _lib.ptr(self.d_ws), self.ws_bytes, _lib.ptr(out), _lib.stream_ptr(stream)),
            "occx_score_topk")
        return out

    def score_partials(self, d_records, n: int, index_base: int = 0, stream=None):
        """K2 only: per-CTA tables left in the workspace (timing / custom merges)."""
        _lib.check(_lib.load().occx_score_topk(
            self._ctx, _lib.ptr(self.h_archs), self.n_arch, _lib.ptr(d_records), n, index_base,
            MODE_CODE[self.mode], _lib.ptr(self.d_vtab), self.n_var, self.n_seg, self.k,
            _lib.ptr(self.d_ws), self.ws_bytes, None, _lib.stream_ptr(stream)),
            "occx_score_topk")
        return self.d_ws

    def score_host(self, host, n: int, index_base: int = 0, chunk: int = 1 << 24):
        """Score n records held in pinned host memory (uint8 tensor, 16 B
        each): chunked H2D on a copy stream, double-buffered against K2 on
        the current stream; per-chunk tables merged by K3.  Returns the
        device [n_seg, k] table (stream-ordered on the current stream)."""
        torch = _torch()
        cur = torch.cuda.current_stream()
        if getattr(self, "_copy_stream", None) is None:
            self._copy_stream = torch.cuda.Stream()
        if getattr(self, "_stage", None) is None or self._stage[0].numel() < chunk * 16:
            self._stage = [_empty(chunk * 16), _empty(chunk * 16)]
        n_chunks = max(1, -(-n // chunk))
        tables = torch.empty((n_chunks, self.n_seg, self.k), dtype=torch.int64, device="cuda")
        freed = [None, None]
        for i in range(n_chunks):
            b = i * chunk
            m = min(chunk, n - b)
            if m <= 0:
                break
            buf = self._stage[i % 2]
            with torch.cuda.stream(self._copy_stream):
                if freed[i % 2] is not None:
                    self._copy_stream.wait_event(freed[i % 2])
                buf[: m * 16].copy_(host[b * 16:(b + m) * 16], non_blocking=True)
                ready = self._copy_stream.record_event()
            cur.wait_event(ready)
            self.score(buf, m, index_base=index_base + b, out=tables[i], stream=cur)
            freed[i % 2] = cur.record_event()
        if n_chunks == 1:
            return tables[0]
        return self.merge(tables, n_chunks)

    def score_implicit(self, begin: int = 0, n: int | None = None, out=None, stream=None,
                       merge: bool = True, key_offset: int = 0, prune: bool = True):
        """K2i: score candidates [begin, begin+n) of the space decoded from their
        global index inside the kernel (no records in HBM).  Identical keys to
        generate() + score(); returns the device [n_seg, k] table.
        ``key_offset`` shifts the index carried in the keys (a weak-scaling
        rank scoring its own copy of the space).  ``prune=False`` evaluates
        every candidate's key (no exact block-bound skipping; same top-k)."""
        torch = _torch()
        n = self.total - begin if n is None else n
        if merge and out is None:
            out = torch.empty((self.n_seg, self.k), dtype=torch.int64, device="cuda")
        _lib.check(_lib.load().occx_score_space(
            self._ctx, _lib.ptr(self.h_archs), self.n_arch, _lib.ptr(self.d_desc), self.n_seg,
            _lib.ptr(self.d_pool), self.n_pool, begin, n, key_offset, MODE_CODE[self.mode],
            0 if prune else _lib.SCORE_EVERY_KEY,
            _lib.ptr(self.d_vtab), self.n_var, self.n_seg, self.k, _lib.ptr(self.d_ws),
            self.ws_bytes, _lib.ptr(out) if merge else None, _lib.stream_ptr(stream)),
            "occx_score_space")
        return out if merge else self.d_ws

    def merge(self, d_lists, n_lists: int, out=None, stream=None):
        """K3 over [n_lists, n_seg, k] device tables -> [n_seg, k]."""
        return merge_tables(d_lists, n_lists, self.n_seg, self.k, out, stream, self._ctx)

    # -- decoding -----------------------------------------------------------
    def locate(self, gidx: int) -> tuple[int, tuple]:
        """Global index -> (segment, enumerate_space tuple of its kernel)."""
        s = bisect.bisect_right(self.seg_start, gidx) - 1
        local = gidx - self.seg_start[s]
        dims = self.seg_dims[s]
        digits = []
        for vals in reversed(dims):
            local, r = divmod(local, len(vals))
            digits.append(vals[r])
        return s, tuple(reversed(digits))

    def decode(self, keys) -> list[SegmentTopK]:
        """[n_seg, k] keys -> per-segment Ranked entries (_SpacePack.decode)."""
        return _SpacePack.decode(self, keys)


def merge_tables(d_lists, n_lists: int, n_seg: int, k: int, out=None, stream=None, ctx=None):
    """K3: [n_lists, n_seg, k] device top-k tables -> merged [n_seg, k]."""
    torch = _torch()
    out = out if out is not None else torch.empty((n_seg, k), dtype=torch.int64, device="cuda")
    _lib.check(_lib.load().occx_topk_merge(
        ctx if ctx is not None else _lib.ctx(), _lib.ptr(d_lists), n_lists, n_seg, k,
        _lib.ptr(out), _lib.stream_ptr(stream)), "occx_topk_merge")
    return out


class ctypes_u64:
    def __init__(self):
        import ctypes
        self._v = ctypes.c_uint64(0)
        self._ctypes = ctypes

    def ref(self):
        return self._ctypes.byref(self._v)

    @property
    def value(self) -> int:
        return int(self._v.value)


def score_space(kernels: Sequence[KernelSpec], archs: Sequence[ArchSpec],
                mode: Mode = Mode.CORRECTED, k: int = 16,
                prune: bool = True) -> list[SegmentTopK]:
    """Score every candidate of the kernels' spaces on every arch; return
    the top-k configurations per (kernel, arch).  Candidates are decoded
    from their index inside the scorer (K2i): nothing but the space
    description, the feature table and the top-k table touch HBM.
    ``prune=False`` evaluates every key (no exact block skipping)."""
    return space_score(_SpacePack(kernels, archs, k), mode, prune=prune)[0]


def space_score(pk: _SpacePack, mode=Mode.CORRECTED, begin: int = 0, n: int | None = None,
                key_offset: int = 0, prune: bool = True, table=DEFAULT_THROUGHPUT,
                scale: float = 1.0, to_host: bool = True):
    """One occx_score_space_host call for a packed space: the description
    goes H2D, K1 + feature table + K2i over [begin, begin+n) + K3 run on the
    current stream.  to_host: returns (decoded segments, u64 keys [n_seg,
    k] host array); else (None, device int64 [n_seg, k] view) without a
    wait (the all-gather path)."""
    torch = _torch()
    n = pk.total - begin if n is None else n
    lib, ctx = _lib.load(), _lib.ctx()
    nb, topk_off = ctypes_u64(), ctypes_u64()
    _lib.check(lib.occx_space_buf_bytes(ctx, len(pk.blob), pk.n_var, pk.n_arch, pk.n_seg,
                                        pk.k, nb.ref(), topk_off.ref()), "occx_space_buf_bytes")
    d_buf = _empty(nb.value)
    h_keys = np.empty((pk.n_seg, pk.k), np.uint64) if to_host else None
    blob_c = (ctypes.c_char * len(pk.blob)).from_buffer(pk.blob)
    _lib.check(lib.occx_score_space_host(
        ctx, pk.h_archs.ctypes.data, pk.n_arch, ctypes.addressof(blob_c), len(pk.blob),
        (ctypes.c_uint64 * 5)(*pk.offsets), pk.n_seg, pk.n_pool, pk.n_var,
        table.cpi_matrix().ctypes.data, float(scale), SUM_MODE, begin, n, key_offset,
        MODE_CODE[Mode(mode)], 0 if prune else _lib.SCORE_EVERY_KEY, pk.k, d_buf.data_ptr(),
        nb.value, h_keys.ctypes.data if to_host else None, _lib.stream_ptr()),
        "occx_score_space_host")
    if to_host:
        return pk.decode(h_keys), h_keys
    off = topk_off.value
    return None, d_buf[off:off + 8 * pk.n_seg * pk.k].view(torch.int64).view(pk.n_seg, pk.k)
