"""One kernel's workload for an ncu capture: three launches of the named
kernel (profile the third: ncu -k regex:NAME -s 2 -c 1).

    python scripts/ncu_workloads.py kd|k1|k3|k4|k0|k0sig

kd  occ_dump_kernel   acceptance-7a sweep, 1,605,632 launches (bench.py)
k1  feature_kernel    the 100k config-3 corpus mixes x 4 cost columns
k3  topk_merge_kernel config 5 K2 partial tables (148 lists x 20 x 16)
k4  suggest_kernel    500k suggest() requests (bench.py secondary)
k0  mix_reduce_kernel config 3, class records (identity class table)
k0sig                 config 3, signature-id records (14,415-entry table)
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1701_08547_b200 import _lib, batch, workloads  # noqa: E402


def main(which):
    if which == "kd":
        import bench
        archs, launches, ai = bench._sweep_7a()
        rec = batch._to_device(batch.pack_launches(launches, ai))
        out = batch._empty(len(launches) * _lib.OCC.itemsize)
        for _ in range(3):
            batch.occupancy_records(archs, rec, len(launches), d_out=out)
    elif which == "k1":
        c = workloads.make_corpus(100_000)
        rec = batch.classify_records(workloads.corpus_records(c), workloads.corpus_signature_lut())
        d = batch.mix_reduce(batch._to_device(rec), batch._to_device(c.offsets), c.n_kernels,
                             batch._to_device(batch.CLASS_LUT), len(batch.CLASS_LUT))
        from paper_1701_08547_b200.mix import DEFAULT_THROUGHPUT
        for _ in range(3):
            batch.feature_records(d, c.n_kernels, [0, 1, 2, 3], DEFAULT_THROUGHPUT.cpi_matrix(), 1.0)
    elif which == "k3":
        cfg = workloads.config5()
        plan = batch.ScorePlan(cfg.kernels, cfg.archs, k=cfg.k)
        n = plan.total
        rec = plan.generate(0, n)
        ws = plan.score_partials(rec, n)
        for _ in range(3):
            plan.merge(ws, plan.grid_lists)
    elif which == "k4":
        from paper_1701_08547_b200.arch import pack_archs
        archs = workloads.all_archs()
        rng = np.random.default_rng(1701)
        nk = 100_000
        inp = np.zeros(nk * len(archs), _lib.SUGG_IN)
        inp["arch"] = np.repeat(np.arange(len(archs)), nk)
        inp["regs"] = np.tile(rng.integers(0, 81, nk), len(archs))
        inp["smem"] = np.tile(rng.integers(0, 48, nk) * 1024, len(archs))
        h = pack_archs(archs)
        d_in, d_out = batch._to_device(inp), batch._empty(len(inp) * _lib.SUGG.itemsize)
        for _ in range(3):
            _lib.check(_lib.load().occx_suggest_batch(_lib.ctx(), _lib.ptr(h), len(h),
                                                      _lib.ptr(d_in), len(inp), 0,
                                                      _lib.ptr(d_out), _lib.stream_ptr()), "k4")
    elif which in ("k0", "k0sig"):
        c = workloads.make_corpus(100_000)
        rec, lut = workloads.corpus_records(c), workloads.corpus_signature_lut()
        if which == "k0":
            rec, lut = batch.classify_records(rec, lut), batch.CLASS_LUT
        d_rec, d_off, d_lut = (batch._to_device(x) for x in (rec, c.offsets, lut))
        out = batch._empty(c.n_kernels * _lib.MIX.itemsize)
        for _ in range(3):
            batch.mix_reduce(d_rec, d_off, c.n_kernels, d_lut, len(lut), d_out=out)
    else:
        raise SystemExit(__doc__)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "")
