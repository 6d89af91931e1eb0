"""Per-kernel analysis reports on the GPU backend.

Mirrors occmix/report.py: ``KernelAnalysis`` (ref report.py:27-42),
``analyze_kernel`` (:45-77), the dict builders ``resources_dict`` ..
``report_dict`` (:89-191) and ``to_json`` (:194-197), so a caller of the
reference gets the same objects and byte-identical JSON.

The difference is where the numbers come from.  ``analyze_batch`` runs the
whole static pipeline for many kernels with one launch per stage:

    K0 mix_reduce       aggregate()                 (all kernels at once)
    K1 feature_score    intensity / cost / cycles / per-class / shares
    K4 suggest          suggest()
    Kd occupancy dump   occupancy() at the suggested launch
    host                static_prune / rule_prune (set logic over <= 32
                        thread counts; tuning.py:94-127)

``analyze_listing`` is the ``occmix analyze`` data path (ref cli.py:105-
134): resource report + disassembly text in, one analysis per resource
stanza out; the listing is tokenized by the native tokenizer (occx_sass)
straight into K0 records.  Errors are raised with the reference's classes
in the reference's order (per kernel: suggest, then cost_estimate, then
the prunes; kernels in input order).
"""

from __future__ import annotations

import enum
import json
import sys
from dataclasses import dataclass, field

import numpy as np

from . import __version__, _lib
from .arch import ArchSpec
from .batch import (FeatureBatch, SignatureTable, _to_device, _to_host, cost_key_of_cc,
                    feature_records, mix_from_record, mix_reduce, occupancy_batch,
                    pack_instructions, suggest_batch, CLASS_LUT)
from .mix import (DEFAULT_OPCLASSES, DEFAULT_THROUGHPUT, InstructionMix, OpClass,
                  category_cycles, per_class_cycles, pipeline_utilization)
from .occupancy import Mode, OccupancyResult, SuggestionReport
from .resources import KernelResources, parse_resource_report
from .tuning import PruneReport, TuningSpace, rule_prune, static_prune

REPORT_FORMAT_VERSION = 1


@dataclass(frozen=True)
class KernelAnalysis:
    """Everything derived for one kernel on one architecture (ref
    report.py:27-42).  ``features`` carries the K1 row the numbers came
    from, so ``kernel_dict`` needs no further launch; it is not part of the
    reference's fields and is excluded from equality."""

    arch: ArchSpec
    mode: Mode
    resources: KernelResources
    mix: InstructionMix
    mix_intensity: float
    cost: float
    suggestion: SuggestionReport
    occupancy_at_best: OccupancyResult
    static_prune: PruneReport
    intensity_prune: PruneReport
    dynamic_shared_mem: int = 0
    scale: float = 1.0
    features: object = field(default=None, compare=False, repr=False)


# ---------------------------------------------------------------------------
# the batched pipeline
# ---------------------------------------------------------------------------

def _pipeline(arch: ArchSpec, resources, d_rec, d_off, n_kernels: int, lut: np.ndarray,
              kernel_of: list, mode: Mode, dynamic_shared_mem: int,
              space: TuningSpace, scale: float) -> list[KernelAnalysis]:
    """K0 over ``n_kernels`` CSR streams (the last one may be the shared
    empty stream), then K1/K4/Kd for resource i on stream kernel_of[i]."""
    mode = Mode(mode)
    n_res = len(resources)
    if n_res == 0:
        return []
    d_mix = mix_reduce(d_rec, d_off, n_kernels, _to_device(lut), len(lut))
    used = sorted(set(kernel_of))
    raw = _to_host(d_mix, _lib.MIX, n_kernels)
    mixes = {k: mix_from_record(raw[k]) for k in used}
    # K1 on the device mix array (all streams; a column for this arch)
    cc = arch.compute_capability
    col = cost_key_of_cc(cc)
    d_sum, d_feat = feature_records(d_mix, n_kernels, [col], DEFAULT_THROUGHPUT.cpi_matrix(),
                                    scale if scale > 0 else 1.0)
    fb = FeatureBatch(_to_host(d_sum, _lib.MIXSUM, n_kernels),
                      _to_host(d_feat, _lib.FEAT, n_kernels), 1,
                      [mixes.get(k) for k in range(n_kernels)], [cc])
    inten = fb.sums["intensity"]
    # K4: suggest for every resource stanza (ref report.py:61-62)
    sugg = suggest_batch([(arch, r, dynamic_shared_mem) for r in resources], mode,
                         raise_first=False)
    bad = [i for i, s in enumerate(sugg) if isinstance(s, Exception)]
    first_bad_suggest = bad[0] if bad else n_res
    # Kd: occupancy at the suggested launch (ref report.py:63-66, :73)
    launches = [(s.best_threads, r.registers_per_thread, r.static_shared_mem + dynamic_shared_mem)
                if not isinstance(s, Exception) else (1, 0, 0)
                for s, r in zip(sugg, resources)]
    occ = occupancy_batch(arch, launches, mode)
    out = []
    for i, res in enumerate(resources):
        if i == first_bad_suggest:
            raise sugg[i]
        k = kernel_of[i]
        if scale <= 0:
            raise ValueError("scale must be positive")          # mix.py:328-329
        feats = fb.one(k, 0)                                    # raises for unsupported cc
        s = sugg[i]
        static = static_prune(space, s)                         # NoCandidatesError
        out.append(KernelAnalysis(
            arch=arch, mode=mode, resources=res, mix=mixes[k],
            mix_intensity=float(inten[k]), cost=feats.cost, suggestion=s,
            occupancy_at_best=occ.result(i), static_prune=static,
            intensity_prune=rule_prune(space, s, float(inten[k])),
            dynamic_shared_mem=dynamic_shared_mem, scale=scale, features=feats))
    return out


def analyze_batch(arch: ArchSpec, items, mode: Mode = Mode.CORRECTED,
                  dynamic_shared_mem: int = 0, space: TuningSpace | None = None,
                  scale: float = 1.0, opclass_table: dict | None = None) -> list[KernelAnalysis]:
    """``[analyze_kernel(arch, res, instrs, ...) for res, instrs in items]``
    with one launch per pipeline stage.  Instructions are any objects with
    the reference ``Instruction`` attributes (duck typed)."""
    items = [(res, list(instrs)) for res, instrs in items]
    if not items:
        return []
    sigs = SignatureTable(opclass_table if opclass_table is not None else DEFAULT_OPCLASSES)
    rec, off = pack_instructions([ins for _, ins in items], sigs)
    return _pipeline(arch, [r for r, _ in items], _to_device(rec if len(rec) else
                                                             np.zeros(1, np.uint32)),
                     _to_device(off), len(items), CLASS_LUT, list(range(len(items))), mode,
                     dynamic_shared_mem, space if space is not None else TuningSpace(), scale)


def analyze_kernel(arch: ArchSpec, resources: KernelResources, instructions,
                   mode: Mode = Mode.CORRECTED, dynamic_shared_mem: int = 0,
                   space: TuningSpace | None = None, scale: float = 1.0,
                   opclass_table: dict | None = None) -> KernelAnalysis:
    """ref report.py:45-77 (a batch of one)."""
    return analyze_batch(arch, [(resources, instructions)], mode, dynamic_shared_mem, space,
                         scale, opclass_table)[0]


def analyze_listing(arch: ArchSpec, resource_report: str, disassembly: str,
                    mode: Mode = Mode.CORRECTED, dynamic_shared_mem: int = 0,
                    space: TuningSpace | None = None, scale: float = 1.0,
                    opclass_table: dict | None = None, warn=None) -> list[KernelAnalysis]:
    """The ``occmix analyze`` pipeline (ref cli.py:105-128) on text inputs:
    one analysis per resource stanza; its instructions are those of the
    listing's function of the same name (the last one when a name repeats,
    as the reference's dict does), or an empty stream with a warning."""
    from .sass import tokenize
    resources = parse_resource_report(resource_report)
    toks = tokenize(disassembly, table=opclass_table if opclass_table is not None
                    else DEFAULT_OPCLASSES)
    by_name = {name: k for k, name in enumerate(toks.names)}
    n_k = len(toks.names)
    kernel_of = []
    for res in resources:
        k = by_name.get(res.entry_name)
        if k is None:
            (warn or (lambda m: print(m, file=sys.stderr)))(
                f"warning: no disassembly for kernel {res.entry_name!r}; "
                f"using an empty instruction stream")
            k = n_k                                  # the shared empty stream
        kernel_of.append(k)
    off = np.concatenate([toks.offsets, toks.offsets[-1:]]).astype(np.uint64)
    rec = toks.records if len(toks.records) else np.zeros(1, np.uint32)
    return _pipeline(arch, resources, _to_device(rec), _to_device(off), n_k + 1, CLASS_LUT,
                     kernel_of, mode, dynamic_shared_mem,
                     space if space is not None else TuningSpace(), scale)


# ---------------------------------------------------------------------------
# dict rendering (fixed field order, ref report.py:80-191)
# ---------------------------------------------------------------------------

def _number(x: float):
    return "inf" if x == float("inf") else x       # JSON has no infinity literal


def _plain(v):
    """Enum -> its value, tuple/list -> list (recursively), else unchanged."""
    if isinstance(v, enum.Enum):
        return v.value
    if isinstance(v, (tuple, list)):
        return [_plain(x) for x in v]
    return v


def _record(obj, layout: str) -> dict:
    """Project ``obj`` onto an ordered JSON object.  ``layout`` lists the
    keys in output order; ``key=attr`` reads a differently named attribute."""
    out = {}
    for item in layout.split():
        key, _, attr = item.partition("=")
        out[key] = _plain(getattr(obj, attr or key))
    return out


# Field order of each object (ref report.py:89-151): part of the format.
_RESOURCES = ("entry_name registers_per_thread static_shared_mem const_mem_banks "
              "spill_loads spill_stores target_cc")
_MIX_TOTALS = "flops mem ctrl reg_operands unclassified total_instructions"
_OCCUPANCY = ("warps_per_block limit_warps limit_regs limit_smem active_blocks "
              "active_warps occupancy limiter mode")
_SUGGESTION = ("thread_candidates registers_used register_headroom smem_budget "
               "best_occupancy best_threads best_blocks")
_PRUNE = "rule=rule_applied original_size pruned_size reduction kept_thread_counts"


def resources_dict(res: KernelResources) -> dict:
    return _record(res, _RESOURCES)


def mix_dict(mix: InstructionMix) -> dict:
    """Non-zero counts in OpClass order, then the category totals."""
    present = {c.value: mix.counts[c] for c in OpClass if mix.counts.get(c)}
    return {"counts": present, **_record(mix, _MIX_TOTALS)}


def occupancy_dict(result: OccupancyResult) -> dict:
    return _record(result, _OCCUPANCY)


def suggestion_dict(sugg: SuggestionReport) -> dict:
    return _record(sugg, _SUGGESTION)


def prune_dict(report: PruneReport) -> dict:
    d = _record(report, _PRUNE)
    if report.intensity is not None:        # rule_prune reports only
        d.update(intensity=_number(report.intensity),
                 intensity_source=report.intensity_source)
    return d


def kernel_dict(analysis: KernelAnalysis) -> dict:
    f = analysis.features
    if f is None:                       # built by hand: one K1 launch
        cc = analysis.arch.compute_capability
        cycles = category_cycles(analysis.mix, cc)
        per_class = per_class_cycles(analysis.mix, cc)
        shares = pipeline_utilization(analysis.mix, cc)
    else:
        cycles, per_class, shares = f.cycles, f.per_class, f.shares
    return {
        "name": analysis.resources.entry_name,
        "resources": resources_dict(analysis.resources),
        "dynamic_shared_mem": analysis.dynamic_shared_mem,
        "instruction_mix": mix_dict(analysis.mix),
        "intensity": _number(analysis.mix_intensity),
        "cost": {
            "total": analysis.cost,
            "scale": analysis.scale,
            "per_category": {c.value: v for c, v in cycles.items()},
            "per_class": {c.value: v for c, v in per_class.items()},
        },
        "pipeline_utilization": {c.value: v for c, v in shares.items()},
        "occupancy": occupancy_dict(analysis.occupancy_at_best),
        "suggestion": suggestion_dict(analysis.suggestion),
        "prune": {
            "static": prune_dict(analysis.static_prune),
            "intensity_rule": prune_dict(analysis.intensity_prune),
        },
    }


def report_dict(arch: ArchSpec, mode: Mode, analyses) -> dict:
    return {
        "tool": "occmix",
        "version": __version__,
        "report_format": REPORT_FORMAT_VERSION,
        "arch": arch.name,
        "compute_capability": arch.compute_capability,
        "mode": Mode(mode).value,
        "kernels": [kernel_dict(a) for a in analyses],
    }


def to_json(report: dict) -> str:
    return json.dumps(report, indent=2) + "\n"


__all__ = ["KernelAnalysis", "analyze_kernel", "analyze_batch", "analyze_listing",
           "resources_dict", "mix_dict", "occupancy_dict", "suggestion_dict", "prune_dict",
           "kernel_dict", "report_dict", "to_json", "REPORT_FORMAT_VERSION"]
