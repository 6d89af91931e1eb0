"""Group an ncu SASS source-page CSV (ncu -i R --page source --csv
--print-source sass) into runs of consecutive lines with the same execution
count: python scripts/sass_regions.py FILE.csv [min_share]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix, isamp, itext = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source")
body = [(i, int(r[ix] or 0), int(r[isamp] or 0), r[itext].strip()) for i, r in enumerate(rows[2:])]
tot = sum(b[1] for b in body)
tots = sum(b[2] for b in body)
runs = []
for i, n, s, t in body:
    if runs and runs[-1][0] == n:
        runs[-1][2] += 1; runs[-1][3] += s; runs[-1][5] = i; runs[-1][6].append(t)
    else:
        runs.append([n, i, 1, s, 0, i, [t]])
mins = float(sys.argv[2]) if len(sys.argv) > 2 else 0.005
print(f"total warp instr {tot}, samples {tots}")
for n, i0, c, s, _, i1, txt in runs:
    if n * c / tot >= mins or s / tots >= mins:
        ops = " ".join(sorted({t.split()[0] if not t.startswith('@') else t.split()[1] for t in txt}))[:150]
        print(f"lines {i0:5d}-{i1:5d} exec {n:9d} x{c:3d} = {n*c/1e6:7.2f}M ({100*n*c/tot:4.1f}%) stall {100*s/tots:4.1f}%  {ops}")
