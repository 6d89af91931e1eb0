"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per kernel the launch count, total / mean time and share of all launches.

usage: python scripts/ncu_launch_summary.py launches.csv out.json "<command>" "<note>"
"""
import csv
import json
import re
import sys

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
head, body = rows[0], rows[1:]
ik, iv = head.index("Kernel Name"), head.index("Metric Value")
agg = {}
for r in body:
    name = re.sub(r"\(.*\)$", "", r[ik]).replace("(int)", "").replace("(bool)", "")
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += float(r[iv].replace(",", "")) / 1e3
total = sum(v[1] for v in agg.values()) or 1.0
out = {"command": sys.argv[3] if len(sys.argv) > 3 else "",
       "note": sys.argv[4] if len(sys.argv) > 4 else "",
       "kernels": [{"kernel": k, "launches": n, "total_us": round(t, 1), "mean_us": round(t / n, 1),
                    "share": round(t / total, 4)}
                   for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])]}
json.dump(out, open(sys.argv[2], "w"), indent=1)
print(json.dumps(out, indent=1))
