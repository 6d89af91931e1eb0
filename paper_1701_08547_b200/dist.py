"""Multi-GPU sharding of a search space.

The candidate space shards by global index: rank g of G scores the
contiguous range ``shard_range(total, g, G)`` (records decoded on its own
device, no data-path collective).  The only exchange is one all-gather of
the fixed-size per-rank top-k table ``[n_seg, k]`` u64 (5 KB for the
benchmark configs) followed by the K3 merge on every rank.  Because every
key embeds its candidate's global index, the merged table is identical for
any G (tests/test_dist.py checks G = 1, 2 with gloo on CPU; the GPU path
runs the same code with NCCL over NVLink).
"""

from __future__ import annotations

from typing import Callable

import numpy as np


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """[begin, end) of rank's contiguous shard; sizes differ by at most one."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    base, extra = divmod(total, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def allgather_merge(local_table, merge: Callable, group=None):
    """All-gather every rank's [n_seg, k] table and merge them.

    ``local_table`` is a torch int64 tensor (u64 keys bit-cast); ``merge``
    maps a stacked [world, n_seg, k] tensor to [n_seg, k] (ScorePlan.merge
    on the GPU).  One collective, fixed size, latency-bound.
    """
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    if world == 1:
        return local_table
    n_seg, k = local_table.shape
    gathered = torch.empty((world * n_seg, k), dtype=local_table.dtype,
                           device=local_table.device)
    dist.all_gather_into_tensor(gathered, local_table.contiguous(), group=group)
    return merge(gathered.view(world, n_seg, k))


def score_space_multi(kernels, archs, mode="corrected", k: int = 16, group=None,
                      scaling: str = "strong", gather_on_host: bool = False,
                      prune: bool = True):
    """The multi-GPU form of ``score_space()`` (the public API a user calls on
    every rank): build the plan from the host-side space description (its
    tables go H2D), score on the device with K2i, all-gather + K3 merge the
    fixed-size top-k tables, read them back and decode.  Returns
    ``(segments, keys)``, identical on every rank.

    ``scaling="strong"``: the ranks split one space by index range.
    ``scaling="weak"``: every rank scores its own copy of the space; copy r
    carries global indices [r*total, (r+1)*total) so keys stay unique.
    ``gather_on_host``: all-gather host tensors (gloo transport).
    ``prune=False``: evaluate every candidate's key (same result)."""
    import torch.distributed as dist
    from .batch import _SpacePack, merge_tables, space_score
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    pk = _SpacePack(kernels, archs, k)
    if scaling == "weak":
        begin, n, key_offset = 0, pk.total, rank * pk.total
    elif scaling == "strong":
        begin, end = shard_range(pk.total, rank, world)
        n, key_offset = end - begin, 0
    else:
        raise ValueError("scaling must be 'strong' or 'weak'")
    if world == 1:
        segs, keys = space_score(pk, mode, begin, n, key_offset, prune=prune)
        return segs, keys
    _, local = space_score(pk, mode, begin, n, key_offset, prune=prune, to_host=False)

    def merge(g):
        return merge_tables(g, g.shape[0], pk.n_seg, pk.k)
    if gather_on_host:
        local = allgather_merge(local.cpu(), lambda g: merge(g.cuda()), group)
    else:
        local = allgather_merge(local, merge, group)
    keys = local.cpu().numpy().view(np.uint64)
    return pk.decode(keys), keys


def score_space_sharded(plan, group=None, records=None, stream=None):
    """Score the plan's whole space across the ranks of ``group``; every
    rank returns the merged [n_seg, k] device table.

    ``records``: optional pre-generated device records of this rank's shard
    (read by K2); otherwise the shard is decoded inside the scorer (K2i).
    """
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    begin, end = shard_range(plan.total, rank, world)
    n = end - begin
    if records is not None:
        local = plan.score(records, n, index_base=begin, stream=stream)
    else:
        local = plan.score_implicit(begin, n, stream=stream)
    if world == 1:
        return local
    return allgather_merge(local, lambda g: plan.merge(g, g.shape[0], stream=stream), group)
