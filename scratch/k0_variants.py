"""K0 variant experiment: time each OCCX_K0 variant on config 3, check bytes equal."""
import os, sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_1701_08547_b200 import workloads, batch, _lib
c = workloads.make_corpus(100_000)
rec = workloads.corpus_records(c)
lut = workloads.corpus_signature_lut()
d_rec = batch._to_device(rec); d_off = batch._to_device(c.offsets); d_lut = batch._to_device(lut)
byts = 4 * c.n_instr + 8 * (c.n_kernels + 1) + 144 * c.n_kernels
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
ref = None
for v in sys.argv[1:] or ["s", "v", "w"]:
    os.environ["OCCX_K0"] = v
    out = batch._empty(c.n_kernels * _lib.MIX.itemsize)
    for _ in range(3):
        batch.mix_reduce(d_rec, d_off, c.n_kernels, d_lut, len(lut), d_out=out)
    torch.cuda.synchronize()
    got = out.cpu().numpy().tobytes()
    if ref is None: ref = got
    same = got == ref
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(20):
        flush.fill_(1)
        e0.record(); batch.mix_reduce(d_rec, d_off, c.n_kernels, d_lut, len(lut), d_out=out); e1.record()
        torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    ms = sorted(ts)[len(ts)//2]
    print(f"K0[{v}] {ms:.4f} ms  {c.n_instr/ms/1e6:.1f} G instr/s  {byts/ms/1e6:.1f} GB/s  frac={byts/ms/1e6/6531.3:.3f} same={same}", flush=True)
