"""Instance sharding across GPUs (one process per GPU).

Instances of a minibatch are independent dataflow graphs, so the hot path shards with
no data-path collective: each rank plans (ed_plan) and executes (ed_execute) its own shard.
Partitioning: LPT by node count — instances sorted by node count descending (ties
by index), each assigned to the currently least-loaded rank (ties to the lowest rank).
"""
from __future__ import annotations

import heapq
from typing import List, Sequence


def lpt_partition(sizes: Sequence[int], world: int) -> List[List[int]]:
    """Instance indices per rank (each rank's list in ascending instance order)."""
    order = sorted(range(len(sizes)), key=lambda i: (-sizes[i], i))
    heap = [(0, r) for r in range(world)]
    heapq.heapify(heap)
    shards: List[List[int]] = [[] for _ in range(world)]
    for i in order:
        load, r = heapq.heappop(heap)
        shards[r].append(i)
        heapq.heappush(heap, (load + max(int(sizes[i]), 1), r))
    return [sorted(s) for s in shards]


def shard_graphs(graphs, rank: int, world: int):
    """(indices, graphs) of this rank's LPT shard."""
    idx = lpt_partition([g.num_nodes for g in graphs], world)[rank]
    return idx, [graphs[i] for i in idx]


def gather_roots(out_local, idx: Sequence[int], n_total: int, group=None):
    """All ranks' root outputs in global instance order (one all-gather of the root
    rows over NCCL / NVLink).  out_local: [len(idx), h] this rank's roots (instance order of idx).
    Every rank contributes a padded [max_shard, h] block plus its instance indices; the result is
    [n_total, h] on every rank.  The only collective of the sharded path (instances are independent,
    P:73)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    n_local = torch.tensor([len(idx)], device=out_local.device)
    sizes = [torch.zeros_like(n_local) for _ in range(world)]
    dist.all_gather(sizes, n_local, group=group)
    cap = int(max(int(s.item()) for s in sizes))
    h = out_local.shape[1]
    pad = torch.zeros(cap, h, dtype=out_local.dtype, device=out_local.device)
    pad[:len(idx)] = out_local
    ids = torch.full((cap,), -1, dtype=torch.int64, device=out_local.device)
    ids[:len(idx)] = torch.as_tensor(list(idx), dtype=torch.int64, device=out_local.device)
    if dist.get_backend(group) == "nccl":
        rows = torch.empty(world * cap, h, dtype=out_local.dtype, device=out_local.device)
        all_ids = torch.empty(world * cap, dtype=torch.int64, device=out_local.device)
        dist.all_gather_into_tensor(rows, pad, group=group)
        dist.all_gather_into_tensor(all_ids, ids, group=group)
    else:
        rl = [torch.empty_like(pad) for _ in range(world)]
        il = [torch.empty_like(ids) for _ in range(world)]
        dist.all_gather(rl, pad, group=group)
        dist.all_gather(il, ids, group=group)
        rows, all_ids = torch.cat(rl), torch.cat(il)
    out = torch.empty(n_total, h, dtype=out_local.dtype, device=out_local.device)
    keep = all_ids >= 0
    out[all_ids[keep]] = rows[keep]
    return out
