"""bench.py's JSON contract: the reference arm on CPU, and (GPU) the
multi-rank path through torchrun with the gloo harness on one device."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout=600, env=None):
    r = subprocess.run([sys.executable, *args], cwd=ROOT, capture_output=True, text=True,
                       timeout=timeout, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run(["bench.py", "--impl", "reference", "--steps", "1", "--warmup", "3",
              "--workload", "config4", "--cpu-sample", "40000"])
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "candidates/s"
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    assert d["higher_is_better"] is True and d["scaling"] == "strong"


def test_self_launch_command(monkeypatch):
    """`bench.py --gpus N` outside torchrun starts N ranks itself (one per
    GPU, rendezvous on 127.0.0.1) with NCCL init logging on."""
    import bench
    seen = {}

    class R:
        returncode = 0

    def fake_run(cmd, env):
        seen["cmd"], seen["env"] = cmd, env
        return R()
    monkeypatch.setattr(subprocess, "run", fake_run)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "5"])
    assert bench.self_launch(4) == 0
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd
    assert cmd[-4:] == ["--gpus", "4", "--steps", "5"] and cmd[-5].endswith("bench.py")
    assert seen["env"]["NCCL_DEBUG"] and seen["env"]["OCCX_BENCH_SELF_LAUNCHED"] == "1"


def test_world_size_must_match_gpus():
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "4"], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=120)
    assert r.returncode != 0 and "--gpus 4 but WORLD_SIZE=2" in r.stderr


@pytest.mark.gpu
def test_self_launched_two_ranks_strong_golden():
    """No torchrun: bench.py launches its 2 ranks itself (gloo harness on the
    one GPU), splits config 2 by index range and checks the merged top-k
    against tests/golden/topk_config2.json on every rank."""
    d = _run(["bench.py", "--gpus", "2", "--steps", "3", "--warmup", "3", "--dist-backend",
              "gloo", "--workload", "config2", "--no-cpu", "--no-secondary"], timeout=900)
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["launch"].startswith("self-launched")
    assert d["topk_equals_golden"] is True
    assert d["config"]["candidates"] == 26_214_400
    assert d["phases_ms"]["allgather_and_k3"] > 0 and len(d["roofline"]["frac_per_rank"]) == 2


@pytest.mark.gpu
@pytest.mark.parametrize("scaling", ["weak", "strong"])
def test_two_rank_bench_line_gloo_harness(scaling):
    d = _run(["-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
              "--master-addr", "127.0.0.1", "--master-port", "29611" if scaling == "weak" else "29612",
              "bench.py", "--gpus", "2", "--steps", "3", "--warmup", "3", "--dist-backend", "gloo",
              "--workload", "config4", "--no-cpu", "--scaling", scaling], timeout=900)
    assert d["n_gpus"] == 2 and d["scaling"] == scaling
    per = d["config"]["candidates_per_gpu"]
    assert d["config"]["candidates"] == (2 * per if scaling == "weak" else 104_857_600)
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] == 3 * 3
    assert d["roofline"]["bound"] == "hbm" and d["clocks"]["sm_max_mhz"]


def test_committed_bench_line_contract():
    """The last GPU bench line committed under profiles/ carries every key of
    the driver contract plus roofline / cpu_baseline / e2e (with the pruned
    library default beside the every-key headline) and in-window clocks."""
    with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                           "profiles", "r01_bench.json")) as fh:
        d = json.loads(fh.read().strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert key in d, key
    assert d["warmup"] >= 3 and d["gpu_launches"] > 0
    r = d["roofline"]
    assert r["bound"] == "hbm" and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert d["cpu_baseline"]["kind"] in ("port", "reference") and d["cpu_baseline"]["cores"] >= 1
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert e["pruned"]["value"] >= e["value"] * 0.9
    assert not set(d["clocks"]["reasons"]) & {"hw_slowdown", "hw_thermal_slowdown",
                                               "sw_thermal_slowdown"}
