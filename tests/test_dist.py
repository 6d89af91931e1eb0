"""Multi-rank sharding on CPU: world_size 2 over gloo.  Every rank scores
its index-range shard with the oracle, the fixed-size top-k tables are
all-gathered through paper_1701_08547_b200.dist.allgather_merge, and the
merged result must equal the single-process golden (G-independence)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from helpers import load_golden
from paper_1701_08547_b200 import workloads
from paper_1701_08547_b200.dist import allgather_merge, shard_range


def test_shard_range_partitions():
    for total in (0, 1, 7, 26_214_400, 1_284_505_600):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_range(total, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [e - b for b, e in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = workloads.CONFIGS[name]()
    prob = oracle.problem_of(cfg)
    b, e = shard_range(cfg.total, rank, world)
    local = oracle.score_spaces(prob, oracle.spaces_of(cfg), b, e, threads=2)
    t = torch.from_numpy(local.view(np.int64).copy())
    merged = allgather_merge(t, lambda g: torch.from_numpy(
        oracle.merge(g.numpy().view(np.uint64), cfg.k).view(np.int64)))
    if rank == 0:
        out.put(merged.numpy().view(np.uint64).tolist())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name,world", [("config2", 2), ("config1", 2), ("config2", 3)])
def test_gloo_sharded_topk_equals_golden(name, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res == load_golden(f"topk_{name}.json")["corrected"]
