"""Report rendering without a GPU: rebuild the value objects from the
reference's own JSON reports (tests/golden/report.json, written by occmix's
report_dict/to_json) and re-render them with this package's dict builders.
Field order, enum values, list conversion and the "inf" spelling must come
out byte-identical (ref report.py:82-151).  The full GPU pipeline is
compared against the same goldens in test_gpu_report.py."""

import json
import os

from paper_1701_08547_b200 import (InstructionMix, KernelResources, Limiter, Mode,
                                   OccupancyResult, OpClass, PruneReport, PruneRule,
                                   SuggestionReport)
from paper_1701_08547_b200.report import (mix_dict, occupancy_dict, prune_dict,
                                          resources_dict, suggestion_dict)

HERE = os.path.dirname(os.path.abspath(__file__))


def _kernels():
    with open(os.path.join(HERE, "golden", "report.json")) as fh:
        g = json.load(fh)
    for run in g["atax"]["runs"]:
        if run["result"]["ok"]:
            yield from json.loads(run["result"]["text"])["kernels"]


def _same(ours, theirs):
    assert json.dumps(ours, indent=2) == json.dumps(theirs, indent=2)


def test_dict_builders_reproduce_reference_json():
    n = 0
    for k in _kernels():
        r = dict(k["resources"])
        r["const_mem_banks"] = tuple(tuple(b) for b in r["const_mem_banks"])
        _same(resources_dict(KernelResources(**r)), k["resources"])

        m = k["instruction_mix"]
        mix = InstructionMix({OpClass(c): v for c, v in m["counts"].items()}, m["reg_operands"])
        _same(mix_dict(mix), m)

        o = dict(k["occupancy"], limiter=Limiter(k["occupancy"]["limiter"]),
                 mode=Mode(k["occupancy"]["mode"]))
        _same(occupancy_dict(OccupancyResult(**o)), k["occupancy"])

        s = dict(k["suggestion"], thread_candidates=tuple(k["suggestion"]["thread_candidates"]))
        _same(suggestion_dict(SuggestionReport(**s)), k["suggestion"])

        for p in k["prune"].values():
            extra = {}
            if "intensity" in p:
                x = p["intensity"]
                extra = dict(intensity=float("inf") if x == "inf" else x,
                             intensity_source=p["intensity_source"])
            rep = PruneReport(p["original_size"], p["pruned_size"],
                              tuple(p["kept_thread_counts"]), PruneRule(p["rule"]), **extra)
            _same(prune_dict(rep), p)
        n += 1
    assert n >= 10
