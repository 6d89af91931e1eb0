"""Digest an ncu --set full report on the box into small files and delete it
(gpurun copies back at most 64 MiB): PREFIX.json (ncu_kernel_summary.py
fields), PREFIX_sass_top.csv (the 80 SASS lines with the most warp
instructions: index, instructions, stall samples, text), PREFIX_ops.json
(warp instructions per opcode).

    python scripts/ncu_digest.py REP.ncu-rep PREFIX --workload W --alg-bytes B \
        [--units U] [--command C] [--note N] [--keep]
"""
import argparse
import collections
import csv
import io
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("prefix")
    ap.add_argument("--workload", required=True)
    ap.add_argument("--alg-bytes", type=float, required=True)
    ap.add_argument("--units", type=float, default=None)
    ap.add_argument("--command", default="")
    ap.add_argument("--note", default="")
    ap.add_argument("--keep", action="store_true")
    a = ap.parse_args()
    cmd = [sys.executable, os.path.join(HERE, "ncu_kernel_summary.py"), a.rep, a.prefix + ".json",
           "--workload", a.workload, "--alg-bytes", str(a.alg_bytes), "--command", a.command,
           "--note", a.note]
    if a.units:
        cmd += ["--units", str(a.units)]
    subprocess.run(cmd, check=True, stdout=subprocess.DEVNULL)
    out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hi = next((i for i, r in enumerate(rows) if "Instructions Executed" in r), None)
    if hi is not None:
        hdr, data = rows[hi], rows[hi + 1:]
        ia, isrc = hdr.index("Instructions Executed"), hdr.index("Source")
        iss = hdr.index("Warp Stall Sampling (All Samples)")
        ops = collections.Counter()
        for r in data:
            t = r[isrc].strip().split()
            if t:
                op = t[1] if t[0].startswith("@") else t[0]
                ops[op.split(".")[0]] += int(r[ia] or 0)
        with open(a.prefix + "_ops.json", "w") as fh:
            json.dump(dict(ops.most_common()), fh, indent=1)
        top = sorted(range(len(data)), key=lambda i: -int(data[i][ia] or 0))[:80]
        with open(a.prefix + "_sass_top.csv", "w", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(["line", "warp_instructions", "stall_samples", "sass"])
            for i in sorted(top):
                w.writerow([i, data[i][ia], data[i][iss], data[i][isrc].strip()])
    if not a.keep:
        os.remove(a.rep)


if __name__ == "__main__":
    main()
