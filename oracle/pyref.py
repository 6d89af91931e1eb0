"""TEST INFRASTRUCTURE ONLY -- pure-Python restatement of the occmix
reference algorithm for the scored hot path.

Used by tests/ as an independent checker for small cases, to derive the
per-(variant, arch) features the C oracle (occx_oracle.c) needs, and by
bench.py's CPU-baseline / ``--impl reference`` leg as "the reference's own
CPU implementation" (the reference is pure Python and cannot travel to the
GPU box, so this line-for-line restatement stands in for it; it is pinned
to the reference by tests/golden fixtures).  Nothing in
paper_1701_08547_b200/ imports this module.

Every function cites the reference line range it restates
(/root/reference/pkg/src/occmix/...).  Floating point uses the running
interpreter's builtin ``sum()``, exactly as the reference does.
"""

from __future__ import annotations

import contextlib
import functools
import heapq
import math
import operator

# CPython's builtin float sum() is Neumaier-compensated from 3.12 on and a
# plain left-to-right loop before (Objects/bltinmodule.c builtin_sum_impl:
# int start 0, then ``f_result += item`` per float).  The reference sums its
# float terms with builtin sum() (mix.py:278, :330, :349), so its bits depend
# on the interpreter; _fsum is the summation every float sum below uses:
# builtin sum() by default, or the <= 3.11 loop under sum_semantics("naive").
_fsum = sum


def naive_sum(values):
    """CPython <= 3.11 float sum(): ((0 + x0) + x1) + ... left to right."""
    return functools.reduce(operator.add, values, 0)


@contextlib.contextmanager
def sum_semantics(which):
    """Restate the reference under another interpreter's sum():
    "naive" (CPython <= 3.11) or "builtin" (this interpreter)."""
    global _fsum
    old = _fsum
    _fsum = {"naive": naive_sum, "builtin": sum}[which]
    try:
        yield
    finally:
        _fsum = old


class OracleIllegalLaunch(Exception):
    """Stands in for occmix.IllegalLaunchError."""


class OracleUnsupported(Exception):
    """Stands in for occmix.UnsupportedArchitectureError."""


# ---------------------------------------------------------------------------
# occupancy.py
# ---------------------------------------------------------------------------

def _ceil_div(a, b):                      # occupancy.py:85-86
    return -(-a // b)


def _round_up(v, g):                      # occupancy.py:89-90
    return _ceil_div(v, g) * g


def warps_per_block(A, t):                # occupancy.py:93-94
    return _ceil_div(t, A.warp_size)


def _check_threads(A, t):                 # occupancy.py:97-101
    if not 1 <= t <= A.max_threads_per_block:
        raise OracleIllegalLaunch(t)


def limit_by_warps(A, t):                 # occupancy.py:104-108
    _check_threads(A, t)
    return min(A.max_blocks_per_mp, A.max_warps_per_mp // warps_per_block(A, t))


def register_warp_limit(A, r):            # occupancy.py:111-124
    if r == 0:
        return A.max_warps_per_mp
    if r > A.max_regs_per_thread:
        return 0
    return A.register_file_size // _round_up(r * A.warp_size,
                                             A.register_alloc_granularity)


def limit_by_registers(A, t, r, verbatim=False):   # occupancy.py:127-145
    _check_threads(A, t)
    if r > A.max_regs_per_thread:
        return 0
    if r == 0:
        return A.max_blocks_per_mp
    wpb = warps_per_block(A, t)
    if verbatim:
        avail = A.register_alloc_granularity // (r * A.warp_size)
        return _ceil_div(avail, wpb) * _ceil_div(A.register_file_size,
                                                 A.register_alloc_granularity)
    return min(A.max_blocks_per_mp, register_warp_limit(A, r) // wpb)


def limit_by_smem(A, s, verbatim=False):  # occupancy.py:148-160
    if s > A.shared_mem_per_block:
        return 0
    if s == 0:
        return A.max_blocks_per_mp
    if verbatim:
        return _ceil_div(A.shared_mem_per_block, s)
    return min(A.max_blocks_per_mp, A.shared_mem_per_block // s)


LIMITERS = ("warps", "registers", "shared-memory", "illegal")


def occupancy(A, t, r=0, s=0, verbatim=False):
    """occupancy.py:38-52 (LaunchInput) + :163-195.  Returns
    (wpb, lw, lr, ls, blocks, active_warps, occupancy, limiter)."""
    if t < 1 or r < 0 or s < 0:
        raise OracleIllegalLaunch(t)
    wpb = warps_per_block(A, t)
    lw = limit_by_warps(A, t)
    lr = limit_by_registers(A, t, r, verbatim)
    ls = limit_by_smem(A, s, verbatim)
    b = min(lw, lr, ls)
    lim = 3 if b == 0 else 0 if b == lw else 1 if b == lr else 2
    aw = min(b * wpb, A.max_warps_per_mp)
    return wpb, lw, lr, ls, b, aw, aw / A.max_warps_per_mp, LIMITERS[lim]


def thread_candidates(A):                 # occupancy.py:198-211
    out = []
    for t in range(A.warp_size, A.max_threads_per_block + 1, A.warp_size):
        wpb = t // A.warp_size
        b = min(A.max_blocks_per_mp, A.max_warps_per_mp // wpb)
        if b >= 1 and wpb * b == A.max_warps_per_mp:
            out.append(t)
    return tuple(out)


def _active_warps_at(A, t, r, s, verbatim):   # occupancy.py:214-229
    wpb = warps_per_block(A, t)
    bound = min(limit_by_warps(A, t) * wpb, A.max_warps_per_mp)
    if verbatim:
        bound = min(bound, limit_by_registers(A, t, r, True) * wpb)
    else:
        bound = min(bound, register_warp_limit(A, r))
    return min(bound, limit_by_smem(A, s, verbatim) * wpb)


def suggest(A, regs, smem, verbatim=False):   # occupancy.py:232-279
    if regs > A.max_regs_per_thread or smem > A.shared_mem_per_block:
        raise OracleIllegalLaunch(regs)
    cands = thread_candidates(A)
    best_t, best_w = cands[0], -1
    for t in cands:
        w = _active_warps_at(A, t, regs, smem, verbatim)
        if w > best_w:
            best_t, best_w = t, w
    wpb = warps_per_block(A, best_t)
    blocks = _ceil_div(best_w, wpb) if best_w else 0
    return {
        "thread_candidates": cands,
        "best_occupancy": best_w / A.max_warps_per_mp,
        "best_threads": best_t,
        "best_blocks": blocks,
        "smem_budget": A.shared_mem_per_block // blocks if blocks else 0,
        "register_headroom": max(0, A.register_file_size // (best_w * A.warp_size) - regs)
        if best_w else 0,
    }


# ---------------------------------------------------------------------------
# tuning.py
# ---------------------------------------------------------------------------

THRESHOLD = 4.0                           # tuning.py:22


def static_kept(thread_counts, cands):    # tuning.py:94-106 (kept tuple)
    return tuple(t for t in thread_counts if t in cands)


def rule_kept(kept, mix_intensity):       # tuning.py:109-127 (kept tuple)
    k = sorted(kept)
    half = -(-len(k) // 2)
    return tuple(k[-half:] if mix_intensity > THRESHOLD else k[:half])


# ---------------------------------------------------------------------------
# mix.py -- classes by their string value
# ---------------------------------------------------------------------------

CLASS_NAMES = ("FPIns32", "FPIns64", "CompMinMax", "ShiftExtractShuffleSAD",
               "Conv64", "Conv32", "LogSinCos", "IntAdd32", "TexIns", "LdStIns",
               "SurfIns", "PredIns", "CtrlIns", "MoveIns", "Unclassified")
CATEGORY = {c: "FLOPS" for c in CLASS_NAMES[:8]}
CATEGORY.update({c: "MEM" for c in CLASS_NAMES[8:11]})
CATEGORY.update({c: "CTRL" for c in CLASS_NAMES[11:14]})
CATEGORY["Regs"] = "REG"

# Table II (mix.py:80-96): class -> IPC for sm20, sm35, sm52, sm60
IPC = {
    "FPIns32": (32, 192, 128, 64), "FPIns64": (16, 64, 4, 32),
    "CompMinMax": (32, 160, 64, 32), "ShiftExtractShuffleSAD": (16, 32, 64, 32),
    "Conv64": (16, 8, 4, 16), "Conv32": (16, 128, 32, 16),
    "LogSinCos": (4, 32, 32, 16), "IntAdd32": (32, 160, 64, 32),
    "TexIns": (16, 32, 64, 16), "LdStIns": (16, 32, 64, 16),
    "SurfIns": (16, 32, 64, 16), "PredIns": (16, 32, 64, 16),
    "CtrlIns": (16, 32, 64, 16), "MoveIns": (32, 32, 32, 32),
    "Regs": (16, 32, 32, 16),
}
_COLUMN = {2: 0, 3: 1, 5: 2, 6: 3}        # mix.py:76, :99-106


def column(cc):
    col = _COLUMN.get(int(cc))
    if col is None:
        raise OracleUnsupported(cc)
    return col


def cpi(cls, col):                        # mix.py:120-124
    return 1.0 / IPC[cls][col]


def _cat_total(counts, cat):              # mix.py:210-211
    return sum(n for c, n in counts.items() if CATEGORY.get(c) == cat)


def flops(counts):
    return _cat_total(counts, "FLOPS")


def mem(counts):
    return _cat_total(counts, "MEM")


def ctrl(counts):
    return _cat_total(counts, "CTRL")


def _flops_coefficient(counts, col):      # mix.py:268-281
    total = flops(counts)
    if total == 0:
        return cpi("FPIns32", col)
    weighted = _fsum([n * cpi(c, col) for c, n in counts.items()
                      if CATEGORY.get(c) == "FLOPS"])
    return weighted / total


def category_cycles(counts, reg_operands, cc):   # mix.py:284-306
    col = column(cc)
    coef = (_flops_coefficient(counts, col), cpi("LdStIns", col),
            cpi("CtrlIns", col), cpi("Regs", col))
    return {"FLOPS": coef[0] * flops(counts), "MEM": coef[1] * mem(counts),
            "CTRL": coef[2] * ctrl(counts), "REG": coef[3] * reg_operands}


def cost_estimate(counts, reg_operands, cc, scale=1.0):   # mix.py:321-330
    if scale <= 0:
        raise ValueError("scale must be positive")
    return scale * _fsum(list(category_cycles(counts, reg_operands, cc).values()))


def intensity(counts):                    # mix.py:333-337
    m = mem(counts)
    if m == 0:
        return math.inf if flops(counts) > 0 else 0.0
    return flops(counts) / m


def pipeline_utilization(counts, reg_operands, cc):   # mix.py:340-352
    cyc = category_cycles(counts, reg_operands, cc)
    total = _fsum(list(cyc.values()))
    if total == 0:
        return {k: 0.0 for k in cyc}
    return {k: v / total for k, v in cyc.items()}


def per_class_cycles(counts, reg_operands, cc):       # mix.py:309-318
    col = column(cc)
    out = {c: n * cpi(c, col) for c, n in counts.items() if c != "Unclassified" and n}
    if reg_operands:
        out["Regs"] = reg_operands * cpi("Regs", col)
    return out


def classify(opcode, modifiers, table):   # mix.py:176-187 (table: key -> class name)
    for m in modifiers:
        hit = table.get(opcode + m)
        if hit is not None:
            return hit
    return table.get(opcode, "Unclassified")


def aggregate(instrs, table):
    """mix.py:245-261.  instrs: iterable of (opcode, modifiers, guarded,
    register_operand_count).  Returns (ordered counts dict, reg_operands)."""
    counts = {}
    regs = 0
    for opcode, mods, guarded, nreg in instrs:
        c = classify(opcode, mods, table)
        counts[c] = counts.get(c, 0) + 1
        if guarded and CATEGORY.get(c) != "CTRL":
            counts["PredIns"] = counts.get("PredIns", 0) + 1
        regs += nreg
    return counts, regs


# ---------------------------------------------------------------------------
# Scoring composition
# ---------------------------------------------------------------------------

IDX_MASK = (1 << 34) - 1


def dense_ranks(costs):
    """Dense rank of each cost among the list (0 = cheapest)."""
    order = sorted(set(costs))
    pos = {c: i for i, c in enumerate(order)}
    return [pos[c] for c in costs]


class Problem:
    """Semantic description the oracle scores, built by the tests from the
    workload definition: archs (ArchSpec-like), kernels each with
    ``thread_counts`` and per-variant (counts dict, reg_operands) mixes."""

    def __init__(self, archs, kernels, verbatim=False, k=16):
        self.archs = list(archs)
        self.kernels = list(kernels)   # [(thread_counts, [(counts, regs), ...]), ...]
        self.verbatim = verbatim
        self.k = k
        self.var_kernel = []
        self.var_mix = []
        for ki, (_, mixes) in enumerate(self.kernels):
            for m in mixes:
                self.var_kernel.append(ki)
                self.var_mix.append(m)
        n_arch = len(self.archs)
        self.n_seg = len(self.kernels) * n_arch
        # per (variant, arch): (seg, rank or -1, upper)
        self.vent = {}
        cands = [frozenset(thread_candidates(A)) for A in self.archs]
        self.sets = {}
        for ki, (tcs, mixes) in enumerate(self.kernels):
            for a, A in enumerate(self.archs):
                st = static_kept(tcs, cands[a])
                self.sets[ki * n_arch + a] = (
                    frozenset(st), frozenset(rule_kept(st, 0.0)) if st else frozenset(),
                    frozenset(rule_kept(st, math.inf)) if st else frozenset())
        for ki in range(len(self.kernels)):
            vs = [v for v, kk in enumerate(self.var_kernel) if kk == ki]
            for a, A in enumerate(self.archs):
                try:
                    column(A.compute_capability)
                    costs = [cost_estimate(*self.var_mix[v], A.compute_capability) for v in vs]
                    ranks = dense_ranks(costs)
                except OracleUnsupported:
                    ranks = [-1] * len(vs)
                for v, rk in zip(vs, ranks):
                    up = intensity(self.var_mix[v][0]) > THRESHOLD
                    self.vent[(v, a)] = (ki * n_arch + a, rk, up)

    def key(self, variant, a, t, r, s, gidx):
        """u64 key of one candidate (0 = illegal / excluded)."""
        if not (0 <= a < len(self.archs)) or not (0 <= variant < len(self.var_kernel)):
            return 0, -1
        try:
            res = occupancy(self.archs[a], t, r, s, self.verbatim)
        except OracleIllegalLaunch:
            return 0, -1
        if res[4] == 0:
            return 0, -1
        seg, rank, up = self.vent[(variant, a)]
        st, lo, hi = self.sets[seg]
        key = (1 << 63) | ((t in (hi if up else lo)) << 62) | ((t in st) << 61) \
            | (res[5] << 54) | ((((1 << 20) - 1 - rank) if rank >= 0 else 0) << 34) \
            | (IDX_MASK - gidx)
        return key, seg


def score_candidates(problem, cands, index_base=0):
    """Composed B0 scorer: cands = iterable of (variant, arch, T, R, S).
    Returns per-segment top-k key lists (descending, 0-padded)."""
    heaps = [[] for _ in range(problem.n_seg)]
    k = problem.k
    for i, (v, a, t, r, s) in enumerate(cands):
        key, seg = problem.key(v, a, t, r, s, index_base + i)
        if key == 0:
            continue
        h = heaps[seg]
        if len(h) < k:
            heapq.heappush(h, key)
        elif key > h[0]:
            heapq.heapreplace(h, key)
    out = []
    for h in heaps:
        lst = sorted(h, reverse=True)
        out.append(lst + [0] * (k - len(lst)))
    return out


def key_index(key):
    """Global candidate index carried in a key's low 34 bits."""
    return IDX_MASK - (key & IDX_MASK)
