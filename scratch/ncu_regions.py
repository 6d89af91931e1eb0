import csv, subprocess, sys
src = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines())); h = rows[1]; data = rows[2:]
ie = h.index("Instructions Executed"); s = h.index("Source"); sp = h.index("Warp Stall Sampling (All Samples)")
prev=None; acc_s=0; acc_i=0; start=0; out=[]
for i,x in enumerate(data):
    n=int(x[ie])
    if n!=prev:
        if prev is not None: out.append((start,i-1,prev,acc_i,acc_s))
        prev=n; acc_s=0; acc_i=0; start=i
    acc_s+=int(x[sp]); acc_i+=n
out.append((start,len(data)-1,prev,acc_i,acc_s))
T=sum(o[3] for o in out); S=sum(o[4] for o in out)
for o in out:
    if o[4]>S*0.01 or o[3]>T*0.01: print(f"{o[0]:5d}-{o[1]:5d} x{o[2]:>8d} inst {o[3]/T*100:5.1f}% samp {o[4]/S*100:5.1f}%  {data[o[0]][s].strip()[:50]}")
