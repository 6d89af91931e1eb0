"""Per-region instruction / stall summary of an ncu source page (SASS).

    python scripts/ncu_regions.py report.ncu-rep [min_executed]

Prints every SASS line executed at least `min_executed` times (default
1e5) with its warp-instruction count and stall samples, plus totals."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 1e5
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = rows[2:]
ia = hdr.index("Instructions Executed")
iss = hdr.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[ia]) for r in data)
stot = sum(int(r[iss]) for r in data)
print(f"total warp instructions {tot}  stall samples {stot}")
for i, r in enumerate(data):
    n = int(r[ia])
    if n >= thr:
        print(f"{i:5d} {n:10d} {int(r[iss]):6d} {r[1][:80]}")
