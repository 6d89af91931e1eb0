import csv, subprocess, sys
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines())); h = rows[0]; r = rows[2]
want = ['gpu__time_duration.sum','dram__bytes_read.sum','sm__warps_active.avg.pct_of_peak_sustained_active','smsp__inst_executed.sum','sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active','smsp__issue_active.avg.pct_of_peak_sustained_active','l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum','l1tex__data_pipe_lsu_wavefronts_mem_shared.sum','launch__registers_per_thread','launch__grid_size','dram__throughput.avg.pct_of_peak_sustained_elapsed']
for w in want:
    if w in h: print(w, r[h.index(w)], rows[1][h.index(w)])
st = [x for x in h if x.startswith('smsp__pcsamp_warps_issue_stalled_') and not x.endswith('not_issued')]
tot = sum(float(r[h.index(x)] or 0) for x in st)
for x in sorted(st, key=lambda x: -float(r[h.index(x)] or 0))[:8]:
    print("  stall", x.replace('smsp__pcsamp_warps_issue_stalled_',''), r[h.index(x)], f"{float(r[h.index(x)])/tot:.2f}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
h = rows[1]; data = rows[2:]
ie = h.index("Instructions Executed"); s = h.index("Source"); sp = h.index("Warp Stall Sampling (All Samples)")
T = sum(int(x[ie]) for x in data); S = sum(int(x[sp]) for x in data)
print("total inst", T, "samples", S)
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.01
for i, x in enumerate(data):
    if int(x[sp]) > S * thr:
        print(f"{i:5d} {x[s].strip()[:64]:64s} {x[ie]:>9s} {x[sp]:>6s}")
