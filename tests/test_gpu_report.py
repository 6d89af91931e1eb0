"""Analysis reports on the GPU (report.py: K0 + K1 + K4 + Kd) against the
reference's own `occmix analyze` JSON, recorded in tests/golden/report.json
by make_golden.py: sha256 of the whole to_json() text and of every kernel
dict, or the exception class and message the reference raised."""

import hashlib
import json

import pytest

from helpers import load_golden, same_sum_semantics
from paper_1701_08547_b200 import (Mode, TuningSpace, analyze_batch, analyze_kernel,
                                   analyze_listing, parse_disassembly, parse_resource_report,
                                   report_dict, to_json, workloads)
from paper_1701_08547_b200.report import kernel_dict

pytestmark = pytest.mark.gpu

SPACES = {"default": None, "verbatim": None,
          "space_scale_dyn": TuningSpace((64, 128, 192, 256, 384, 512, 1024), (8, 16), (1, 2),
                                         (16, 48), ("", "-O3"))}
PARAMS = {"default": ("corrected", 1.0, 0), "verbatim": ("verbatim", 1.0, 0),
          "space_scale_dyn": ("corrected", 2.5, 1024)}


@pytest.fixture(scope="module")
def g():
    g = load_golden("report.json")
    if not same_sum_semantics(g["meta"]):
        pytest.skip("report floats recorded under another CPython sum()")
    return g


def _run(arch, case, res_text, sass_text):
    mode, scale, dyn = PARAMS[case]
    try:
        an = analyze_listing(arch, res_text, sass_text, Mode(mode), dynamic_shared_mem=dyn,
                             space=SPACES[case], scale=scale, warn=lambda m: None)
    except Exception as exc:   # noqa: BLE001
        return {"ok": False, "error": type(exc).__name__, "message": str(exc)}, None
    text = to_json(report_dict(arch, Mode(mode), an))
    return {"ok": True, "sha256": hashlib.sha256(text.encode()).hexdigest(),
            "kernels": [hashlib.sha256(json.dumps(kernel_dict(a), indent=2).encode())
                        .hexdigest()[:16] for a in an]}, text


def _check(got, want, text=None):
    if not want["ok"]:
        assert (got.get("error"), got.get("message")) == (want["error"], want["message"])
        return
    assert got["ok"], got
    if want.get("text") is not None and text != want["text"]:
        import difflib
        diff = "".join(list(difflib.unified_diff(want["text"].splitlines(True),
                                                 text.splitlines(True)))[:40])
        pytest.fail("report JSON differs from the reference:\n" + diff)
    bad = [i for i, (a, b) in enumerate(zip(got["kernels"], want["kernels"])) if a != b]
    assert not bad and len(got["kernels"]) == len(want["kernels"]), bad[:5]
    assert got["sha256"] == want["sha256"]


def test_atax_reports_byte_identical(g):
    archs = workloads.all_archs()
    for run in g["atax"]["runs"]:
        got, text = _run(archs[run["arch"]], run["case"], g["atax"]["ptxas"], g["atax"]["sass"])
        _check(got, run["result"], text)


def test_corpus_reports_byte_identical(g):
    archs = workloads.all_archs()
    c = workloads.make_corpus(g["n_kernels"])
    sass = workloads.corpus_text(c)
    assert hashlib.sha256(sass.encode()).hexdigest() == g["sass_sha256"]
    for run in g["corpus"]:
        a = archs[run["arch"]]
        dyn = PARAMS[run["case"]][2]
        res = workloads.corpus_resource_report(g["n_kernels"], run["seed"], a.max_regs_per_thread,
                                               a.shared_mem_per_block - dyn)
        got, _ = _run(a, run["case"], res, sass)
        _check(got, run["result"])


def test_error_paths_match_reference(g):
    kepler = workloads.all_archs()[1]
    sass = workloads.corpus_text(workloads.make_corpus(g["n_kernels"]))
    for case in g["errors"]:
        try:
            analyze_listing(kepler, case["resources"], sass, scale=case["scale"],
                            warn=lambda m: None)
            got = {"ok": True}
        except Exception as exc:   # noqa: BLE001
            got = {"ok": False, "error": type(exc).__name__, "message": str(exc)}
        _check(got, case["result"])


def test_object_api_equals_listing_api(g):
    """analyze_kernel / analyze_batch on parsed Instruction objects give the
    same report as the tokenizer path."""
    kepler = workloads.all_archs()[1]
    (res,) = parse_resource_report(g["atax"]["ptxas"])
    ((_, ins),) = parse_disassembly(g["atax"]["sass"])
    one = analyze_kernel(kepler, res, ins)
    want = next(r["result"] for r in g["atax"]["runs"] if r["arch"] == 1 and r["case"] == "default")
    assert to_json(report_dict(kepler, Mode.CORRECTED, [one])) == want["text"]
    many = analyze_batch(kepler, [(res, ins)] * 3 + [(res, [])])
    assert [to_json(kernel_dict(a)) for a in many[:3]] == [to_json(kernel_dict(one))] * 3
    assert many[3].mix.total_instructions == 0
