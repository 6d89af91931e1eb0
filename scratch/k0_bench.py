import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_1701_08547_b200 import workloads, batch, _lib
t0 = time.time()
c = workloads.make_corpus(100_000)
rec = workloads.corpus_records(c)
lut = workloads.corpus_signature_lut()
print("gen", time.time() - t0, c.n_instr)
d_rec = batch._to_device(rec); d_off = batch._to_device(c.offsets); d_lut = batch._to_device(lut)
out = batch._empty(c.n_kernels * _lib.MIX.itemsize)
for _ in range(3):
    batch.mix_reduce(d_rec, d_off, c.n_kernels, d_lut, len(lut), d_out=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
ts = []
for _ in range(10):
    flush.fill_(1)
    e0.record(); batch.mix_reduce(d_rec, d_off, c.n_kernels, d_lut, len(lut), d_out=out); e1.record()
    torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
ms = sorted(ts)[len(ts)//2]
byts = 4 * c.n_instr + 8 * (c.n_kernels + 1) + 144 * c.n_kernels
print(f"K0 {ms:.3f} ms  {c.n_instr/ms/1e6:.1f} G instr/s  {byts/ms/1e6:.1f} GB/s  frac={byts/ms/1e6/6531.3:.3f}")
