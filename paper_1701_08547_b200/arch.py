"""Architecture database: per-SM hardware limits (mirrors occmix/arch.py).

Same public surface as the reference -- ``Family``, frozen ``ArchSpec``
(field order and invariants of arch.py:29-81), ``BUILTIN_ARCHS``
(arch.py:84-129), ``builtin_arch`` (:132-143), the INI loader
(:146-204) and ``resolve_arch`` (:207-223).  On top of that every spec
can be packed into the 40-byte ``occx_arch_t`` record the sm_100a
kernels read (include/occx.h); ``device_limits_ok`` states the few
capacity limits of that packed form (all real GPUs satisfy them).
"""

from __future__ import annotations

import configparser
import enum
import io
from dataclasses import dataclass, fields

import numpy as np

from .errors import ArchSpecError, ParseError, UnknownArchitectureError


class Family(str, enum.Enum):
    FERMI = "fermi"
    KEPLER = "kepler"
    MAXWELL = "maxwell"
    PASCAL = "pascal"
    OTHER = "other"


# The ten fields every formula consumes; they must all be > 0.
_POSITIVE = ("multiprocessors", "warp_size", "max_threads_per_mp",
             "max_threads_per_block", "max_blocks_per_mp", "max_warps_per_mp",
             "register_file_size", "register_alloc_granularity",
             "max_regs_per_thread", "shared_mem_per_block")


@dataclass(frozen=True)
class ArchSpec:
    """Per-multiprocessor limits of one GPU generation (immutable)."""

    name: str
    family: Family
    compute_capability: float
    multiprocessors: int
    warp_size: int
    max_threads_per_mp: int
    max_threads_per_block: int
    max_blocks_per_mp: int
    max_warps_per_mp: int
    register_file_size: int
    register_alloc_granularity: int
    max_regs_per_thread: int
    shared_mem_per_block: int
    cuda_cores_per_mp: int | None = None
    global_mem_mb: int | None = None
    gpu_clock_mhz: int | None = None
    mem_clock_mhz: int | None = None
    l2_cache_mb: float | None = None
    constant_mem_bytes: int | None = None

    def __post_init__(self):
        bad = [f for f in _POSITIVE if getattr(self, f) <= 0]
        if bad:
            raise ArchSpecError(bad[0], "must be strictly positive")
        if self.max_threads_per_block % self.warp_size:
            raise ArchSpecError(
                "max_threads_per_block",
                f"{self.max_threads_per_block} is not a multiple of warp_size "
                f"{self.warp_size}")
        if self.max_warps_per_mp * self.warp_size != self.max_threads_per_mp:
            raise ArchSpecError(
                "max_warps_per_mp",
                f"max_warps_per_mp ({self.max_warps_per_mp}) x warp_size "
                f"({self.warp_size}) must equal max_threads_per_mp "
                f"({self.max_threads_per_mp})")
        if self.max_regs_per_thread > self.register_file_size:
            raise ArchSpecError("max_regs_per_thread",
                                "exceeds the register file size")


def _spec(name, family, cc, sms, tpm, bpm, wpm, rfs, gran, rmax, extra):
    """Compact constructor for the built-in table (warp size 32, 1024-thread
    blocks and 48 KiB shared memory are common to all four generations)."""
    cores, gmem, gclk, mclk, l2 = extra
    return ArchSpec(name=name, family=family, compute_capability=cc,
                    multiprocessors=sms, warp_size=32, max_threads_per_mp=tpm,
                    max_threads_per_block=1024, max_blocks_per_mp=bpm,
                    max_warps_per_mp=wpm, register_file_size=rfs,
                    register_alloc_granularity=gran, max_regs_per_thread=rmax,
                    shared_mem_per_block=49152, cuda_cores_per_mp=cores,
                    global_mem_mb=gmem, gpu_clock_mhz=gclk, mem_clock_mhz=mclk,
                    l2_cache_mb=l2, constant_mem_bytes=65536)


# Values of the reference's built-in descriptors (arch.py:84-129).
BUILTIN_ARCHS: dict[Family, ArchSpec] = {
    Family.FERMI: _spec("fermi-m2050", Family.FERMI, 2.0, 14, 1536, 8, 48,
                        32768, 64, 63, (32, 3072, 1147, 1546, 0.786)),
    Family.KEPLER: _spec("kepler-k20", Family.KEPLER, 3.5, 13, 2048, 16, 64,
                         65536, 256, 255, (192, 11520, 824, 2505, 1.572)),
    Family.MAXWELL: _spec("maxwell-m40", Family.MAXWELL, 5.2, 24, 2048, 32, 64,
                          65536, 256, 255, (128, 12288, 1140, 5000, 3.146)),
    Family.PASCAL: _spec("pascal-p100", Family.PASCAL, 6.0, 56, 2048, 32, 64,
                         65536, 256, 255, (64, 17066, 405, 715, 4.194)),
}


def _builtin_names() -> list[str]:
    return [f.value for f in BUILTIN_ARCHS]


def builtin_arch(family: Family | str) -> ArchSpec:
    """Built-in descriptor for a family (ref arch.py:132-143)."""
    if isinstance(family, str):
        try:
            family = Family(family.lower())
        except ValueError:
            raise UnknownArchitectureError(family, _builtin_names())
    if family not in BUILTIN_ARCHS:
        raise UnknownArchitectureError(family.value, _builtin_names())
    return BUILTIN_ARCHS[family]


_INI_REQUIRED = ("family", "compute_capability", "multiprocessors", "warp_size",
                 "max_threads_per_mp", "max_threads_per_block",
                 "max_blocks_per_mp", "max_warps_per_mp", "register_file_size",
                 "register_alloc_granularity", "max_regs_per_thread",
                 "shared_mem_per_block")
_INI_OPTIONAL_INT = ("cuda_cores_per_mp", "global_mem_mb", "gpu_clock_mhz",
                     "mem_clock_mhz", "constant_mem_bytes")


def _section_to_spec(name: str, sec) -> ArchSpec:
    missing = [k for k in _INI_REQUIRED if k not in sec]
    if missing:
        raise ArchSpecError(missing[0], f"missing in section [{name}]")
    try:
        family = Family(sec["family"].lower())
    except ValueError:
        family = Family.OTHER
    kw: dict = {"name": name, "family": family}
    for key in _INI_REQUIRED[1:]:
        text = sec[key]
        try:
            kw[key] = float(text) if key == "compute_capability" else int(text)
        except ValueError:
            raise ArchSpecError(key, f"not a number: {text!r}")
    kw.update({k: int(sec[k]) for k in _INI_OPTIONAL_INT if k in sec})
    if "l2_cache_mb" in sec:
        kw["l2_cache_mb"] = float(sec["l2_cache_mb"])
    return ArchSpec(**kw)


def parse_arch_config(text: str) -> list[ArchSpec]:
    """Parse INI text into specs, atomically (ref arch.py:170-181)."""
    cp = configparser.ConfigParser()
    try:
        cp.read_file(io.StringIO(text))
    except configparser.ParsingError as exc:
        raise ParseError(f"bad config syntax: {exc.message.splitlines()[0]}",
                         exc.errors[0][0] if exc.errors else None)
    except configparser.Error as exc:
        raise ParseError(f"bad config syntax: {exc}")
    return [_section_to_spec(s, cp[s]) for s in cp.sections()]


def load_arch_file(path: str) -> list[ArchSpec]:
    """Read an INI architecture database (ref arch.py:146-167)."""
    with open(path, encoding="utf-8") as fh:
        return parse_arch_config(fh.read())


def resolve_arch(name: str, user_specs: list[ArchSpec] = ()) -> ArchSpec:
    """User specs (by name) shadow built-ins (by name or family) (ref arch.py:207-223)."""
    wanted = name.lower()
    for spec in user_specs:
        if spec.name.lower() == wanted:
            return spec
    for spec in BUILTIN_ARCHS.values():
        if wanted == spec.name or wanted == spec.family.value:
            return spec
    known = {s.name for s in user_specs}
    known |= {s.name for s in BUILTIN_ARCHS.values()}
    known |= {s.family.value for s in BUILTIN_ARCHS.values()}
    raise UnknownArchitectureError(name, sorted(known))


# ---------------------------------------------------------------------------
# Packing for the device (occx_arch_t, include/occx.h)
# ---------------------------------------------------------------------------

# cost column of the Table II throughput data, keyed by int(cc); ref mix.py:76
COST_KEY_OF_MAJOR = {2: 0, 3: 1, 5: 2, 6: 3}

ARCH_DTYPE = np.dtype([
    ("warp_size", "<i4"), ("max_threads_per_block", "<i4"),
    ("max_blocks_per_mp", "<i4"), ("max_warps_per_mp", "<i4"),
    ("register_file_size", "<i4"), ("register_alloc_granularity", "<i4"),
    ("max_regs_per_thread", "<i4"), ("shared_mem_per_block", "<i4"),
    ("cost_key", "<i4"), ("reserved", "<i4"),
])
assert ARCH_DTYPE.itemsize == 40


def cost_key(spec: ArchSpec) -> int:
    """Throughput-table column index, or -1 when the reference raises
    UnsupportedArchitectureError (ref mix.py:99-106)."""
    return COST_KEY_OF_MAJOR.get(int(spec.compute_capability), -1)


def device_limits_ok(spec: ArchSpec) -> str | None:
    """None when the packed form can represent ``spec`` exactly, else why not.

    Limits of the device tables (hold for every shipped NVIDIA GPU); the
    same set ``occx_check_archs`` (csrc/occx_score.cu) enforces, so an arch
    either fails here with its field named or is accepted by every kernel:
    power-of-two warp size, <= 64 warps per block, at most 2048 threads
    per block (the static / rule membership masks hold bit T/32 - 1 < 64;
    every warp-size-32 arch fits), <= 1023
    registers per thread, <= 255 blocks and <= 127 warps per SM (u8 / 7-bit
    key fields), register file and allocation granularity below 2**20,
    shared memory below 2**24 bytes.
    """
    ws = spec.warp_size
    if ws <= 0 or ws & (ws - 1):
        return "warp_size must be a power of two"
    if spec.max_threads_per_block // ws > 64:
        return "more than 64 warps per block"
    if spec.max_threads_per_block > 2048:
        return "max_threads_per_block above 2048 (membership masks cover T <= 2048)"
    if spec.max_regs_per_thread > 1023:
        return "max_regs_per_thread above 1023"
    if spec.max_blocks_per_mp > 255:
        return "max_blocks_per_mp above 255"
    if spec.max_warps_per_mp > 127:
        return "max_warps_per_mp above 127"
    if spec.shared_mem_per_block >= 1 << 24:
        return "shared_mem_per_block at or above 2**24"
    if spec.register_file_size >= 1 << 20:
        return "register_file_size at or above 2**20"
    if spec.register_alloc_granularity >= 1 << 20:
        return "register_alloc_granularity at or above 2**20"
    return None


def pack_archs(specs) -> np.ndarray:
    """Pack specs into an ``occx_arch_t`` array; raises ArchSpecError when a
    spec exceeds the device table limits."""
    out = np.zeros(len(specs), dtype=ARCH_DTYPE)
    for i, s in enumerate(specs):
        why = device_limits_ok(s)
        if why:
            raise ArchSpecError(s.name, why)
        for f in ARCH_DTYPE.names[:8]:
            out[i][f] = getattr(s, f)
        out[i]["cost_key"] = cost_key(s)
    return out


SPEC_FIELDS = tuple(f.name for f in fields(ArchSpec))
