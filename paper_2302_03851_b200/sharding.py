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
