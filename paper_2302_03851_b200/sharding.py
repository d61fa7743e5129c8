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


class RootGather:
    """The root all-gather of the sharded path, set up once per plan.

    Construction (outside any timed region) exchanges the shard sizes and instance ids once and
    builds a padded [cap, h] send block and a static index map.  ed_execute writes this rank's roots
    straight into ``local`` (a contiguous view of the send block), so a step is exactly one
    all_gather_into_tensor of the padded blocks plus one index_select into global instance order:
    no host sync, no size exchange, no H2D (sizes are static per plan)."""

    def __init__(self, idx: Sequence[int], n_total: int, h: int, dtype, device, group=None):
        import torch
        import torch.distributed as dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.nccl = dist.get_backend(group) == "nccl"
        dev = torch.device(device)
        cdev = dev if self.nccl else torch.device("cpu")
        n_local = torch.tensor([len(idx)], dtype=torch.int64, device=cdev)
        sizes = [torch.zeros_like(n_local) for _ in range(self.world)]
        dist.all_gather(sizes, n_local, group=group)
        self.cap = cap = max(1, int(max(int(s.item()) for s in sizes)))
        ids = torch.full((cap,), -1, dtype=torch.int64, device=cdev)
        ids[:len(idx)] = torch.as_tensor(list(idx), dtype=torch.int64)
        il = [torch.empty_like(ids) for _ in range(self.world)]
        dist.all_gather(il, ids, group=group)
        all_ids = torch.cat(il).cpu()
        src = torch.full((n_total,), -1, dtype=torch.int64)
        pos = torch.nonzero(all_ids >= 0).flatten()
        src[all_ids[pos]] = pos
        if bool((src < 0).any()):
            raise ValueError("RootGather: the shards do not cover every instance")
        self.src = src.to(dev)
        self.send = torch.zeros(cap, h, dtype=dtype, device=dev)
        self.local = self.send[:len(idx)]
        self.rows = torch.empty(self.world * cap, h, dtype=dtype, device=dev)

    def __call__(self):
        """[n_total, h] roots of every rank in global instance order."""
        import torch
        import torch.distributed as dist
        if self.nccl:
            dist.all_gather_into_tensor(self.rows, self.send, group=self.group)
        else:
            rl = list(torch.chunk(self.rows, self.world))
            dist.all_gather(rl, self.send, group=self.group)
        return self.rows.index_select(0, self.src)


def gather_roots(out_local, idx: Sequence[int], n_total: int, group=None):
    """All ranks' root outputs in global instance order (one-off convenience wrapper over
    RootGather; a timed loop builds the RootGather once and reuses it)."""
    rg = RootGather(idx, n_total, out_local.shape[1], out_local.dtype, out_local.device, group)
    rg.local.copy_(out_local)
    return rg()
