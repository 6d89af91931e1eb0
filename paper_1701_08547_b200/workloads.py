"""Synthetic workloads of BASELINE.json's five configurations.

Inputs only -- no scoring logic.  Shared by bench.py, the tests and the
golden-fixture generator so every arm scores the same candidates.

* kernels: the paper's ATAX (mix of the reference's ATAX fixture,
  tests/data/atax_kepler.sass.txt, R=27), BiCG, MatVec2D and ex14FJ
  (synthetic mixes calibrated to the Table V intensities 1.8 / 4.6 / 12.7,
  PAPER.md:505-527).  Variant (UIF u, CFLAGS f): counts x u; fast math
  moves u FP32 instructions to LogSinCos.
* archs: Fermi, Kepler, Maxwell, Pascal (built-ins) + an sm_100 INI table.
* the 100k-kernel SASS corpus of config 3 (splitmix64, seed 0x170108547),
  emitted both as 4-byte records and, for small subsets, as listing text in
  the reference's grammar (pkg/README.md:152-167).
"""

from __future__ import annotations

from dataclasses import dataclass
from itertools import combinations

import numpy as np

from .arch import BUILTIN_ARCHS, Family, parse_arch_config
from .batch import KernelSpec
from .mix import DEFAULT_OPCLASSES, InstructionMix, OpClass, classify_signature, DEVICE_ID
from .tuning import TuningSpace

SM100_INI = """\
[sm100-b200]
family = other
compute_capability = 10.0
multiprocessors = 148
warp_size = 32
max_threads_per_mp = 2048
max_threads_per_block = 1024
max_blocks_per_mp = 32
max_warps_per_mp = 64
register_file_size = 65536
register_alloc_granularity = 256
max_regs_per_thread = 255
shared_mem_per_block = 232448
"""


def sm100():
    return parse_arch_config(SM100_INI)[0]


def all_archs():
    """Config 2/4/5 arch tables: Fermi, Kepler, Maxwell, Pascal, sm_100."""
    return [BUILTIN_ARCHS[Family.FERMI], BUILTIN_ARCHS[Family.KEPLER],
            BUILTIN_ARCHS[Family.MAXWELL], BUILTIN_ARCHS[Family.PASCAL], sm100()]


_C = OpClass
# (ordered class counts, reg_operands, registers/thread)
BASE_MIXES = {
    # aggregate() of the reference's ATAX fixture (pinned by tests/golden)
    "atax": ([(_C.MOVE, 7), (_C.INT_ADD32, 12), (_C.COMP_MIN_MAX, 2), (_C.CONTROL, 4),
              (_C.LOAD_STORE, 5), (_C.FP32, 3)], 63, 27),
    "bicg": ([(_C.MOVE, 6), (_C.INT_ADD32, 6), (_C.COMP_MIN_MAX, 1), (_C.CONTROL, 4),
              (_C.LOAD_STORE, 5), (_C.FP32, 2)], 48, 24),
    "matvec2d": ([(_C.MOVE, 8), (_C.INT_ADD32, 14), (_C.COMP_MIN_MAX, 2), (_C.CONTROL, 5),
                  (_C.LOAD_STORE, 5), (_C.FP32, 7)], 70, 32),
    "ex14fj": ([(_C.MOVE, 12), (_C.INT_ADD32, 15), (_C.COMP_MIN_MAX, 4), (_C.FP64, 8),
                (_C.CONTROL, 6), (_C.LOAD_STORE, 10), (_C.FP32, 100), (_C.PREDICATE, 3)],
               410, 63),
}
KERNEL_NAMES = tuple(BASE_MIXES)


def variant_mix(name: str, unroll: int, flag: str) -> InstructionMix:
    counts, regs, _ = BASE_MIXES[name]
    d = {c: n * unroll for c, n in counts}
    if flag == "-use_fast_math":
        d[_C.FP32] -= unroll
        d[_C.LOG_SIN_COS] = d.get(_C.LOG_SIN_COS, 0) + unroll
    return InstructionMix(d, regs * unroll)


def kernel_spec(name: str, space: TuningSpace) -> KernelSpec:
    mixes = tuple(variant_mix(name, u, f) for u in space.unroll_factors
                  for f in space.compiler_flags)
    return KernelSpec(name, space, mixes, registers_per_thread=BASE_MIXES[name][2])


@dataclass(frozen=True)
class Config:
    name: str
    kernels: tuple
    archs: tuple
    k: int = 16

    @property
    def total(self) -> int:
        from .tuning import grid_size
        return sum(grid_size(kk.space) for kk in self.kernels) * len(self.archs)


def config1() -> Config:
    """ATAX on Kepler, T 32..1024/32, one variant, R=27, S=0 (32 candidates)."""
    space = TuningSpace(tuple(range(32, 1025, 32)), (24,), (1,), (16,), ("",))
    return Config("config1-atax-kepler", (kernel_spec("atax", space),),
                  (BUILTIN_ARCHS[Family.KEPLER],))


def _grid_config(name, regs, smem) -> Config:
    space = TuningSpace(extra=(("REGS", tuple(regs)), ("SMEM", tuple(smem))))
    return Config(name, tuple(kernel_spec(n, space) for n in KERNEL_NAMES), tuple(all_archs()))


def config2() -> Config:
    """4 kernels x 5 archs, TuningSpace() x R 0..255 x S {0}: 26,214,400."""
    return _grid_config("config2-paper-kernels-full-grid", range(0, 256), (0,))


def config4() -> Config:
    """10^8 space: R 0..255/8 x S 0..49152/1536 per segment: 104,857,600."""
    return _grid_config("config4-1e8-orio-space", range(0, 256, 8), range(0, 49152, 1536))


def config5() -> Config:
    """10^9 space: R 0..255 x S 0..49152/1024 per segment: 1,284,505,600."""
    return _grid_config("config5-1e9-orio-space", range(0, 256), range(0, 49153, 1024))


CONFIGS = {"config1": config1, "config2": config2, "config4": config4, "config5": config5}


# ---------------------------------------------------------------------------
# Config 3: synthetic SASS corpus
# ---------------------------------------------------------------------------

CORPUS_SEED = 0x170108547
MODIFIERS = (".E", ".F64", ".S64", ".U64", ".GE", ".AND", ".FTZ", ".X")
UNIFORM_OPS = ("UIADD3", "ULOP3", "LDCU", "S2UR", "UISETP", "HFMA2", "UMOV", "R2UR",
               "UPRMT", "ULEA")
UNKNOWN_OPS = ("QUUX", "FROB", "WEIRDOP", "ZAP2", "BLORP", "XYZZY", "PLUGH", "GLORK",
               "SNARF", "WIBBLE")
# subsets of MODIFIERS with 0..3 members, canonical order
MOD_SUBSETS = tuple(tuple(MODIFIERS[i] for i in c)
                    for n in range(4) for c in combinations(range(8), n))
_SUBSET_BASE = (0, 1, 9, 37)          # first subset index of each size
_SUBSET_COUNT = (1, 8, 28, 56)
assert len(MOD_SUBSETS) == 93


def corpus_opcodes() -> tuple[str, ...]:
    roots = sorted({k.split(".")[0] for k in DEFAULT_OPCLASSES})
    return tuple(roots) + UNIFORM_OPS + UNKNOWN_OPS


def _splitmix64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


@dataclass
class Corpus:
    offsets: np.ndarray      # u64[n_kernels + 1]
    opcode: np.ndarray       # u16 per instruction (index into corpus_opcodes())
    subset: np.ndarray       # u8  per instruction (index into MOD_SUBSETS)
    guard: np.ndarray        # u8  0 none / 1 "@P0" / 2 "@!P1"
    ops: np.ndarray          # u8[n, 4] operand template ids (255 = none)

    @property
    def n_kernels(self) -> int:
        return len(self.offsets) - 1

    @property
    def n_instr(self) -> int:
        return int(self.offsets[-1])


# operand templates: (text pattern, register occurrences)
OPERAND_TEMPLATES = (("R{a}", 1), ("RZ", 0), ("P{p}", 0), ("c[0x0][0x{c:x}]", 0),
                     ("[R{a}]", 1), ("[R{a}+0x{c:x}]", 1), ("0x{c:x}", 0), ("SR_TID.X", 0))
_REGS_OF_TEMPLATE = np.array([t[1] for t in OPERAND_TEMPLATES] + [0] * 248, np.uint8)


def make_corpus(n_kernels: int = 100_000, seed: int = CORPUS_SEED, first: int = 0) -> Corpus:
    """Kernels [first, first+n_kernels) of the config-3 corpus."""
    kid = np.arange(first, first + n_kernels, dtype=np.uint64)
    hk = _splitmix64(kid ^ np.uint64(seed))
    lengths = (np.uint64(32) + hk % np.uint64(1985)).astype(np.int64)
    offsets = np.zeros(n_kernels + 1, np.uint64)
    np.cumsum(lengths, out=offsets[1:])
    n = int(offsets[-1])
    # instruction i of kernel k hashes (k << 16 | i): independent of `first`
    kern_of = np.repeat(np.arange(n_kernels, dtype=np.uint64), lengths)
    pos = np.arange(n, dtype=np.uint64) - np.repeat(offsets[:-1], lengths)
    h1 = _splitmix64(((kern_of + np.uint64(first)) << np.uint64(16)) ^ pos ^
                     (np.uint64(seed) << np.uint64(40)))
    h2 = _splitmix64(h1)
    n_ops = len(corpus_opcodes())
    n_roots = n_ops - len(UNIFORM_OPS) - len(UNKNOWN_OPS)
    r = (h1 % np.uint64(1000)).astype(np.int64)
    pick = ((h1 >> np.uint64(10)) % np.uint64(1 << 20)).astype(np.int64)
    opcode = np.where(r < 900, pick % n_roots,
                      np.where(r < 950, n_roots + pick % len(UNIFORM_OPS),
                               n_roots + len(UNIFORM_OPS) + pick % len(UNKNOWN_OPS)))
    nmod = ((h1 >> np.uint64(32)) % np.uint64(4)).astype(np.int64)
    base = np.asarray(_SUBSET_BASE)[nmod]
    cnt = np.asarray(_SUBSET_COUNT)[nmod]
    subset = base + ((h1 >> np.uint64(36)) % np.uint64(1 << 16)).astype(np.int64) % cnt
    gr = ((h1 >> np.uint64(54)) % np.uint64(100)).astype(np.int64)
    guard = np.where(gr < 15, 1 + (gr & 1), 0)
    nopnd = (h2 % np.uint64(5)).astype(np.int64)
    ops = np.full((n, 4), 255, np.uint8)
    for j in range(4):
        t = ((h2 >> np.uint64(8 + 3 * j)) & np.uint64(7)).astype(np.uint8)
        ops[:, j] = np.where(nopnd > j, t, 255)
    return Corpus(offsets, opcode.astype(np.uint16), subset.astype(np.uint8),
                  guard.astype(np.uint8), ops)


def corpus_signature_lut(table=DEFAULT_OPCLASSES) -> np.ndarray:
    """u8 class id per signature id = opcode * 93 + subset (classify())."""
    ops = corpus_opcodes()
    lut = np.zeros(len(ops) * len(MOD_SUBSETS), np.uint8)
    for o, name in enumerate(ops):
        for s, mods in enumerate(MOD_SUBSETS):
            lut[o * len(MOD_SUBSETS) + s] = DEVICE_ID[classify_signature(name, mods, table)]
    return lut


def corpus_records(c: Corpus) -> np.ndarray:
    """4-byte instruction records (include/occx.h OCCX_INSTR)."""
    sig = c.opcode.astype(np.uint32) * np.uint32(len(MOD_SUBSETS)) + c.subset.astype(np.uint32)
    regops = _REGS_OF_TEMPLATE[c.ops].sum(axis=1).astype(np.uint32)
    guard = (c.guard > 0).astype(np.uint32)
    return guard | (sig << np.uint32(1)) | (regops << np.uint32(17))


def corpus_text(c: Corpus, kernels=None) -> str:
    """Disassembly listing of some kernels in the reference grammar."""
    ops = corpus_opcodes()
    lines = []
    for k in (range(c.n_kernels) if kernels is None else kernels):
        lines.append(f"\tFunction : kern_{k:06d}")
        for i in range(int(c.offsets[k]), int(c.offsets[k + 1])):
            parts = []
            if c.guard[i]:
                parts.append("@P0" if c.guard[i] == 1 else "@!P1")
            parts.append(ops[c.opcode[i]] + "".join(MOD_SUBSETS[c.subset[i]]))
            opnds = []
            for j, t in enumerate(c.ops[i]):
                if t == 255:
                    break
                opnds.append(OPERAND_TEMPLATES[t][0].format(a=(i + j) % 64, p=j % 7,
                                                            c=(i * 8 + j * 4) % 0x400))
            body = " ".join(parts)
            if opnds:
                body += " " + ", ".join(opnds)
            addr = (i - int(c.offsets[k])) * 16
            lines.append(f"        /*{addr:04x}*/                   {body} ;")
    return "\n".join(lines) + "\n"


def corpus_resource_report(n_kernels: int, seed: int, rmax: int, smax: int) -> str:
    """Synthetic ptxas -v report for corpus kernels kern_000000..: every
    7th name is absent from the listing (empty stream + warning), one name
    repeats, clauses vary (smem, cmem banks, spills, lmem)."""
    import random
    rng = random.Random(seed)
    lines = ["ptxas info    : 0 bytes gmem"]
    names = [f"kern_{k:06d}" for k in range(n_kernels)]
    names[::7] = [f"missing_{k}" for k in range(len(names[::7]))]
    names.append(names[3])
    for i, name in enumerate(names):
        sm = rng.choice(("20", "35", "52", "60", "100a", None))
        lines.append(f"ptxas info    : Compiling entry function '{name}'" +
                     (f" for 'sm_{sm}'" if sm else ""))
        if rng.random() < 0.2:
            lines.append(f"ptxas info    : Function properties for {name}")
            lines.append(f"    {rng.randrange(0, 64)} bytes stack frame, "
                         f"{rng.randrange(0, 9)} bytes spill stores, "
                         f"{rng.randrange(0, 9)} bytes spill loads")
        clauses = [f"{rng.randrange(0, rmax + 1)} registers"]
        if rng.random() < 0.6:
            clauses.append(f"{rng.choice((0, 4, 1024, 3072, 6144, 12288, smax))} bytes smem")
        if rng.random() < 0.8:
            clauses.append(f"{rng.randrange(320, 400)} bytes cmem[0]")
        if rng.random() < 0.2:
            clauses.append(f"{rng.randrange(0, 64)} bytes cmem[2]")
        if rng.random() < 0.1:
            clauses.append("8 bytes lmem")
        lines.append("ptxas info    : Used " + ", ".join(clauses))
    return "\n".join(lines) + "\n"
