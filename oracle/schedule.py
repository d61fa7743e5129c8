"""FSM-based dynamic batching (PAPER Alg. 1) and its comparators — oracle, test infrastructure only.

Alg. 1:
    while G.notEmpty():
        nextType = pi(E(G))
        batch = [v for v in Frontier(G) if v.type is nextType]
        Execute batch; Update the Frontier.

Readings: E_sort orders frontier types by descending frontier count, ties by
ascending type id (A-2); the FSM transition table maps an E_sort key to a type (A-3); on a
table miss, or when the action has no ready node, the fallback is key[0] (A-3).  Batches are
compared as member SETS (A-4); members are listed in ascending global id.

The frontier here is recomputed naively from its definition after every batch (P:123
"Frontier(G) refers to the set of ready-to-execute operations"), independent of the C++
incremental counters.
"""
from __future__ import annotations

import itertools
from typing import Callable, Dict, List, Optional, Sequence, Tuple

from .graph import Merged, topo_depth, typed_subgraph_edges

Schedule = List[Tuple[int, List[int]]]  # (type, sorted members)


def frontier(m: Merged, executed: Sequence[bool]) -> List[int]:
    """All unexecuted nodes whose node inputs are all executed."""
    return [v for v in range(m.n)
            if not executed[v] and all(executed[u] for u in m.node_inputs(v))]


def type_counts(m: Merged, front: Sequence[int]) -> Dict[int, int]:
    c: Dict[int, int] = {}
    for v in front:
        c[m.type[v]] = c.get(m.type[v], 0) + 1
    return c


# --- state encodings -------------------------------------------------------------------

def e_base(counts: Dict[int, int]) -> tuple:
    """E_base(G) = {v.type | v in Frontier(G)} (as a sorted tuple)."""
    return tuple(sorted(counts))


def e_max(counts: Dict[int, int]) -> tuple:
    """E_max(G) = (E_base(G), argmax_t |Frontier_t(G)|), count ties to the lowest type id."""
    best = min(counts, key=lambda t: (-counts[t], t))
    return (e_base(counts), best)


def e_sort(counts: Dict[int, int]) -> tuple:
    """E_sort(G): frontier types sorted by occurrence count (descending; ties ascending id)."""
    return tuple(sorted(counts, key=lambda t: (-counts[t], t)))


ENCODERS = {"sort": e_sort, "base": e_base, "max": e_max}


def all_sort_keys(num_types: int) -> List[tuple]:
    """Every possible E_sort key: non-empty ordered tuples of distinct type ids."""
    keys = []
    for k in range(1, num_types + 1):
        keys.extend(itertools.permutations(range(num_types), k))
    return keys


def table_from_priority(priority: Sequence[int], num_types: int) -> Dict[tuple, int]:
    """Harness convenience (SURVEY A-3): action = highest-priority type present in the key."""
    rank = {t: i for i, t in enumerate(priority)}
    return {key: min(key, key=lambda t: rank.get(t, len(rank) + t)) for key in all_sort_keys(num_types)}


# --- Alg. 1 -----------------------------------------------------------------------------------

def run_alg1(m: Merged, choose: Callable[[Merged, List[bool], List[int], Dict[int, int]], int]) -> Schedule:
    executed = [False] * m.n
    sched: Schedule = []
    while not all(executed):
        front = frontier(m, executed)
        counts = type_counts(m, front)
        t = choose(m, executed, front, counts)
        batch = sorted(v for v in front if m.type[v] == t)
        if not batch:
            raise RuntimeError("chooser returned a type with no ready node")
        for v in batch:
            executed[v] = True
        sched.append((t, batch))
    return sched


def fsm_chooser(table: Dict[tuple, int], encoder: str = "sort") -> Callable:
    """pi(E(G)) by table lookup ("a lookup into stored Q functions"), with the A-3
    fallback key[0] of the E_sort key on a miss or an action that has no ready node."""
    enc = ENCODERS[encoder]

    def choose(m, executed, front, counts):
        key = enc(counts)
        a = table.get(key)
        if a is None or counts.get(a, 0) == 0:
            return e_sort(counts)[0]
        return a
    return choose


def fsm_schedule(m: Merged, table: Dict[tuple, int], encoder: str = "sort") -> Schedule:
    return run_alg1(m, fsm_chooser(table, encoder))


# --- comparators -----------------------------------------------------------------

def depth_schedule(m: Merged) -> Schedule:
    """TF-Fold depth-based batching: one batch per (depth, type) group, groups in
    ascending depth, ties by ascending type id (SPEC S:139 reading)."""
    depth = topo_depth(m)
    groups: Dict[tuple, List[int]] = {}
    for v in range(m.n):
        groups.setdefault((depth[v], m.type[v]), []).append(v)
    return [(t, sorted(groups[(d, t)])) for (d, t) in sorted(groups)]


def agenda_chooser(m: Merged) -> Callable:
    """DyNet agenda-based batching: the ready type with minimal average topological
    depth.  The average runs over ALL nodes of the type (executed included), which is what
    reproduces P:107's "(1+2+3)/3=2" for I after I1 has run (SURVEY A-22); ties by type id."""
    depth = topo_depth(m)
    mean = {}
    for t in range(m.num_types):
        ds = [depth[v] for v in range(m.n) if m.type[v] == t]
        mean[t] = sum(ds) / len(ds) if ds else float("inf")

    def choose(mm, executed, front, counts):
        return min(counts, key=lambda t: (mean[t], t))
    return choose


def readiness_ratio(m: Merged, executed: Sequence[bool], a: int) -> float:
    """Second term of Eq. 1 under the A-1 reading (P:129 display inverted to match the worked
    values 5/7, 1/1 of P:138 and Lemma 1): |Frontier_a(G_t)| / |Frontier(G^a_t)|, where G^a_t is
    the typed subgraph over the UNEXECUTED type-a nodes and its frontier is the set of its nodes
    with no unexecuted type-a predecessor in G^a."""
    front = frontier(m, executed)
    ready_a = [v for v in front if m.type[v] == a]
    nodes_a = [v for v in range(m.n) if m.type[v] == a and not executed[v]]
    has_pred = set()
    for u, w in typed_subgraph_edges(m, a):
        if not executed[u] and not executed[w]:
            has_pred.add(w)
    front_a = [v for v in nodes_a if v not in has_pred]
    return len(ready_a) / len(front_a)


def sc_chooser() -> Callable:
    """Sufficient-condition heuristic: argmax of Eq. 1's second term; ties by the larger
    ready count, then ascending type id (SPEC S:149 reading)."""
    def choose(m, executed, front, counts):
        return min(counts, key=lambda t: (-readiness_ratio(m, executed, t), -counts[t], t))
    return choose


# --- exact optimum and table enumeration (App. B.1 / BJ "brute-force optimal policies") ---------

def optimal_batches(m: Merged, first: Optional[int] = None, limit: int = 48) -> int:
    """Length of the shortest batch-type sequence (App. B.1): breadth-first search over the
    executed-set states reachable by Alg. 1 moves (batch ALL ready nodes of a chosen type).
    ``first`` constrains the first batch's type (Lemma 1 test)."""
    if m.n > limit:
        raise ValueError("graph too large for brute force")
    preds = [m.node_inputs(v) for v in range(m.n)]
    full = (1 << m.n) - 1

    def moves(state):
        ready: Dict[int, int] = {}
        for v in range(m.n):
            if not (state >> v) & 1 and all((state >> u) & 1 for u in preds[v]):
                ready[m.type[v]] = ready.get(m.type[v], 0) | (1 << v)
        return ready

    if m.n == 0:
        return 0
    start = 0
    level = {start}
    seen = {start}
    steps = 0
    while level:
        steps += 1
        nxt = set()
        for s in level:
            mv = moves(s)
            for t, bits in mv.items():
                if steps == 1 and first is not None and t != first:
                    continue
                ns = s | bits
                if ns == full:
                    return steps
                if ns not in seen:
                    seen.add(ns)
                    nxt.add(ns)
        level = nxt
    raise RuntimeError("unreachable")


def enumerate_sort_tables(num_types: int):
    """All E_sort FSM tables: for every key of length >= 2 choose one of its types (single-type
    keys are forced).  4 tables for 2 types, 46,656 for 3."""
    keys = [k for k in all_sort_keys(num_types) if len(k) >= 2]
    for choice in itertools.product(*keys):
        table = {(t,): t for t in range(num_types)}
        table.update(dict(zip(keys, choice)))
        yield table


def validate_schedule(m: Merged, sched: Schedule) -> int:
    """Replay a schedule: homogeneous batches, every node exactly once, no node
    before its inputs.  Returns the batch count; raises AssertionError otherwise."""
    done = [False] * m.n
    for t, members in sched:
        assert members, "empty batch"
        for v in members:
            assert m.type[v] == t, f"node {v} of type {m.type[v]} in a type-{t} batch"
            assert not done[v], f"node {v} issued twice"
            for u in m.node_inputs(v):
                assert done[u], f"node {v} issued before its input {u}"
        for v in members:
            done[v] = True
    assert all(done), "schedule misses nodes"
    return len(sched)
