"""Summarise one kernel of an ncu --set full report into a small JSON file
(the numbers the DESIGN/bench roofline lines cite).

usage: python scripts/ncu_kernel_summary.py REP.ncu-rep OUT.json \
           --workload W --alg-bytes N [--units U] [--command CMD] [--note TEXT]
"""
import argparse
import csv
import json
import subprocess


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(out.splitlines()))
    head, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(head, units, vals)}


def num(m, key, scale=1.0):
    v, u = m[key]
    v = float(str(v).replace(",", ""))
    mult = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "usecond": 1e-3,
            "msecond": 1.0, "nsecond": 1e-6, "us": 1e-3, "ms": 1.0, "ns": 1e-6}.get(u, 1.0)
    return v * mult * scale


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("out")
    ap.add_argument("--workload", required=True)
    ap.add_argument("--alg-bytes", type=float, required=True)
    ap.add_argument("--units", type=float, default=None, help="work units per launch")
    ap.add_argument("--command", default="")
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    m = raw_metrics(a.rep)
    rd = num(m, "dram__bytes_read.sum")
    wr = num(m, "dram__bytes_write.sum")
    ms = num(m, "gpu__time_duration.sum")
    inst = num(m, "smsp__inst_executed.sum")
    stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): num(m, k) for k in m
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
    tot = sum(stalls.values()) or 1.0
    top = sorted(stalls.items(), key=lambda kv: -kv[1])[:6]
    s = {
        "kernel": m["Kernel Name"][0] if "Kernel Name" in m else "",
        "workload": a.workload,
        "command": a.command,
        "duration_ms": ms,
        "dram_bytes_read": rd,
        "dram_bytes_write": wr,
        "dram_bytes_per_launch": rd + wr,
        "algorithmic_bytes_per_launch": a.alg_bytes,
        "achieved_algorithmic_gbs": a.alg_bytes / ms / 1e6,
        "issue_active_pct": num(m, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "alu_pipe_pct": num(m, "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
        "warps_active_pct": num(m, "sm__warps_active.avg.pct_of_peak_sustained_active"),
        "warp_instructions": inst,
        "registers": num(m, "launch__registers_per_thread"),
        "grid": num(m, "launch__grid_size"),
        "block": num(m, "launch__block_size"),
        "smem_wavefronts": num(m, "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
        "smem_bank_conflicts": num(m, "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
        "stall_top": {k: round(v / tot, 3) for k, v in top},
        "note": a.note,
    }
    if a.units:
        s["units_per_launch"] = a.units
        s["thread_instructions_per_unit"] = inst * 32 / a.units
    with open(a.out, "w") as f:
        json.dump(s, f, indent=1)
    print(json.dumps(s, indent=1))


if __name__ == "__main__":
    main()
