"""Merged dataflow DAG and its plain graph quantities (oracle; test infrastructure only).

PAPER.md P:73 (§2.1): "given a mini-batch of input instances, dataflow graphs are generated
for each of the input instances ... and each operation is given a type".  A minibatch is the
disjoint union of the instance graphs (SURVEY A-24); global ids are instance-major prefix
sums of local ids (SURVEY A-5).  Raw inputs (external ids, the zero state) are not
schedulable nodes (SURVEY A-6): only node inputs create dependencies.
"""
from __future__ import annotations

from typing import List, Sequence

import numpy as np


class Merged:
    """Disjoint union of instance graphs with global node ids.

    inputs[v]  list of slot entries: ('n', u) node input u (global id), ('z', 0) zero state,
               ('x', id) external input id.
    """

    def __init__(self, graphs: Sequence, num_types: int):
        self.num_types = num_types
        self.type: List[int] = []
        self.inputs: List[List[tuple]] = []
        self.ext: List[int] = []
        self.instance: List[int] = []
        self.local: List[int] = []
        self.base: List[int] = []
        self.roots: List[tuple] = []
        off = 0
        for gi, g in enumerate(graphs):
            self.base.append(off)
            n = int(g.type.shape[0])
            for v in range(n):
                self.type.append(int(g.type[v]))
                ins = []
                for x in g.in_idx[g.in_off[v]:g.in_off[v + 1]]:
                    x = int(x)
                    if x >= 0:
                        ins.append(("n", off + x))
                    elif x == -(2 ** 31):
                        ins.append(("z", 0))
                    else:
                        ins.append(("x", -1 - x))
                self.inputs.append(ins)
                self.ext.append(int(g.ext[v]))
                self.instance.append(gi)
                self.local.append(v)
            r = int(g.root)
            self.roots.append(("n", off + r) if r >= 0 else ("x", -1 - r))
            off += n
        self.n = off

    def node_inputs(self, v: int) -> List[int]:
        """Distinct dependency predecessors of v (node inputs only)."""
        return sorted({u for k, u in self.inputs[v] if k == "n"})

    def consumers(self) -> List[List[int]]:
        out: List[List[int]] = [[] for _ in range(self.n)]
        for v in range(self.n):
            for u in self.node_inputs(v):
                out[u].append(v)
        return out

    def topo_order(self) -> List[int]:
        """Kahn's algorithm; raises ValueError on a cycle."""
        indeg = [len(self.node_inputs(v)) for v in range(self.n)]
        cons = self.consumers()
        ready = [v for v in range(self.n) if indeg[v] == 0]
        order = []
        while ready:
            v = ready.pop()
            order.append(v)
            for w in cons[v]:
                indeg[w] -= 1
                if indeg[w] == 0:
                    ready.append(w)
        if len(order) != self.n:
            raise ValueError("cycle")
        return order


def topo_depth(m: Merged) -> List[int]:
    """PAPER P:107 "the input operation to the network has depth 0": raw inputs are depth 0,
    an op's depth is 1 + max depth of its node inputs (an op fed only by raw inputs has depth 1,
    reproducing Fig. 1's (1+1+1+1+2+3+4)/7)."""
    depth = [0] * m.n
    for v in m.topo_order():
        depth[v] = 1 + max([depth[u] for u in m.node_inputs(v)], default=0)
    return depth


def typed_subgraph_edges(m: Merged, a: int) -> List[tuple]:
    """Edges of G^a ("the extracted subgraph of G composed solely of type a
    operations"; SURVEY A-21 / SPEC S:48: u->v kept iff G has a path u ~> v whose intermediate
    nodes are all non-a).  Plain definition: a DFS from every a-node through non-a nodes."""
    cons = m.consumers()
    edges = []
    for u in range(m.n):
        if m.type[u] != a:
            continue
        seen = set()
        stack = list(cons[u])
        while stack:
            w = stack.pop()
            if w in seen:
                continue
            seen.add(w)
            if m.type[w] == a:
                edges.append((u, w))
            else:
                stack.extend(cons[w])
    return edges


def longest_path_nodes(nodes: Sequence[int], edges: Sequence[tuple]) -> int:
    """Longest path (counted in nodes) of a DAG given as a node list and an edge list."""
    nodes = list(nodes)
    if not nodes:
        return 0
    succ = {v: [] for v in nodes}
    indeg = {v: 0 for v in nodes}
    for u, w in edges:
        succ[u].append(w)
        indeg[w] += 1
    best = {v: 1 for v in nodes}
    ready = [v for v in nodes if indeg[v] == 0]
    while ready:
        v = ready.pop()
        for w in succ[v]:
            best[w] = max(best[w], best[v] + 1)
            indeg[w] -= 1
            if indeg[w] == 0:
                ready.append(w)
    return max(best.values())


def typed_depth(m: Merged, a: int) -> int:
    """Depth(G^a): longest node path of the typed subgraph (App. B.3, SURVEY A-21)."""
    nodes = [v for v in range(m.n) if m.type[v] == a]
    return longest_path_nodes(nodes, typed_subgraph_edges(m, a))


def lower_bound(m: Merged) -> int:
    """App. B.3 Eq.: |Batching*(G)| >= sum_t Depth(G_t)."""
    return sum(typed_depth(m, a) for a in range(m.num_types))


def lower_bound_dp(m: Merged) -> int:
    """Same quantity by a one-pass DP (count of a-nodes on the best path ending at v); used
    only to cross-check typed_depth on large graphs where the DFS definition is slow."""
    order = m.topo_order()
    total = 0
    for a in range(m.num_types):
        cnt = [0] * m.n
        for v in order:
            cnt[v] = (1 if m.type[v] == a else 0) + max([cnt[u] for u in m.node_inputs(v)], default=0)
        total += max(cnt, default=0)
    return total


def as_numpy_types(m: Merged) -> np.ndarray:
    return np.asarray(m.type, dtype=np.int32)
