"""Memory-layout side of the oracle (PAPER §3; App. C) — test infrastructure only.

Layout variables (SURVEY A-9, a departure from the paper which plans only static subgraphs,
P:262): one variable per node; its output record (h row, c row, MV-RNN matrix) lives at one
row index in parallel buffers.  A layout is row_of_node[v]; the all-zero row (ZERO_INPUT
reads) is row V.

Operands of a batch b: the result operand R_b = the members in position
order, and for each fixed slot j the source operand S_{b,j} = slot-j inputs of the members in
the same positions ("aligned").  Position order of a batch is ascending result row (A-11).
"""
from __future__ import annotations

from typing import Dict, List, Sequence, Tuple

from .graph import Merged


def schedule_order_layout(m: Merged, sched) -> List[int]:
    """ED_LAYOUT_SCHEDULE_ORDER: rows assigned batch after batch (every result operand is then one
    contiguous block, SURVEY A-9); inside a batch, members ordered by
      1. the latest batch that produces one of their node inputs (-1 if none; reading L-1),
      2. their earliest consumer: (consumer's batch, consumer's position inside its batch), the
         smallest over the consumers; members without a consumer after all others (reading L-3),
      3. global id.
    Positions are fixed from the last batch backwards (a consumer's position is known before its
    producers are ordered); then rows are the batches' positions offset by the earlier batches."""
    batch_of = {}
    for b, (_, members) in enumerate(sched):
        for v in members:
            batch_of[v] = b
    consumers = m.consumers()
    pos = {}
    for b in range(len(sched) - 1, -1, -1):
        members = sched[b][1]

        def key(v):
            latest = max([batch_of[u] for u in m.node_inputs(v)], default=-1)
            earliest = min([(batch_of[w], pos[w]) for w in consumers[v]], default=(float("inf"), 0))
            return (latest, earliest, v)
        for k, v in enumerate(sorted(members, key=key)):
            pos[v] = k
    row = [-1] * m.n
    r = 0
    for _, members in sched:
        for v in members:
            row[v] = r + pos[v]
        r += len(members)
    assert r == m.n and sorted(row) == list(range(m.n))
    return row


def batch_positions(members: Sequence[int], row: Sequence[int]) -> List[int]:
    """Members of a batch in position order = ascending result row."""
    return sorted(members, key=lambda v: row[v])


def source_operand(m: Merged, ordered: Sequence[int], slot: int) -> List[tuple]:
    return [m.inputs[v][slot] if slot < len(m.inputs[v]) else None for v in ordered]


def fixed_slots(m: Merged, ordered: Sequence[int]) -> int:
    return min(len(m.inputs[v]) for v in ordered)


def contig_base(entries: Sequence, row: Sequence[int]) -> int:
    """Row base if the operand's rows are base+i for position i (all node inputs), else -1."""
    if not entries or any(e is None or e[0] != "n" for e in entries):
        return -1
    base = row[entries[0][1]]
    for i, e in enumerate(entries):
        if row[e[1]] != base + i:
            return -1
    return base


def check_ideal(m: Merged, sched, row: Sequence[int], fixed_only: int = 99) -> List[Dict]:
    """Per batch (PAPER P:163-167 ideal layout = adjacency + alignment): whether the result
    operand is one contiguous ascending block and, for each fixed slot, whether the source
    operand occupies consecutive ascending rows aligned with the result positions."""
    rep = []
    for t, members in sched:
        ordered = batch_positions(members, row)
        res_ok = all(row[ordered[i]] == row[ordered[0]] + i for i in range(len(ordered)))
        ns = min(fixed_slots(m, ordered), fixed_only)
        srcs = [contig_base(source_operand(m, ordered, j), row) >= 0 for j in range(ns)]
        rep.append({"type": t, "result": res_ok, "sources": srcs})
    return rep


def paper_copy_kernels(m: Merged, sched, row: Sequence[int]) -> Tuple[int, int]:
    """Gather/scatter kernels a DyNet-style executor needs: for each batch pick the
    member permutation pi (taken from the result operand's memory order or from one source
    operand's) that minimises copies; every operand not consecutive-ascending under pi costs one
    kernel — a gather for a source, a scatter for the result.  Ties prefer fewer scatters.
    Returns (gathers, scatters) summed over batches."""
    G = S = 0
    for _, members in sched:
        members = list(members)
        ns = fixed_slots(m, members)
        ops = [[("n", v) for v in members]] + [source_operand(m, members, j) for j in range(ns)]
        # operands reading external rows / the zero state are not layout variables (A-9)
        ops = [o for o in ops if all(e is not None and e[0] == "n" for e in o)]
        best = None
        for ref in ops:
            if any(e is None or e[0] != "n" for e in ref):
                continue
            perm = sorted(range(len(members)), key=lambda i: row[ref[i][1]])
            g = s = 0
            for k, op in enumerate(ops):
                ok = contig_base([op[i] for i in perm], row) >= 0
                if not ok:
                    if k == 0:
                        s += 1
                    else:
                        g += 1
            cand = (g + s, s, g)
            if best is None or cand < best:
                best = cand
        G += best[2]
        S += best[1]
    return G, S


def executor_copy_split(m: Merged, sched, row: Sequence[int]) -> Tuple[int, int]:
    """Gather / scatter kernels of an executor that orders each batch's members by the memory
    position of their slot-0 source (PAPER Fig. 3(b): B1 is written [x4, x5] = alpha([x1, x3],
    [x2, x1]) and B2 [x8, x6, x7] = sigma([x3, x4, x5]) -- in both batches the members follow their
    first source operand; reading A-25b).  A member whose slot-0 input is not a node keeps
    its result position.  Under that order every source operand that is not consecutive-ascending in
    memory costs one gather, a result operand that is not costs one scatter.  Returns (gathers,
    scatters)."""
    G = S = 0
    for _, members in sched:
        members = list(members)
        ns = fixed_slots(m, members)

        def key(v):
            ins = m.inputs[v]
            if ins and ins[0][0] == "n":
                return (0, row[ins[0][1]], row[v])
            return (1, row[v], row[v])
        ordered = sorted(members, key=key)
        if contig_base([("n", v) for v in ordered], row) < 0:
            S += 1
        for j in range(ns):
            op = source_operand(m, ordered, j)
            if all(e is not None and e[0] == "n" for e in op) and contig_base(op, row) < 0:
                G += 1
    return G, S


def copy_bytes(m: Merged, sched, row: Sequence[int], row_bytes: int) -> Tuple[int, int]:
    """Bytes a DyNet-style executor would move (SURVEY §8(d) "bytes avoided"): 2 x rows x
    row_bytes per non-contiguous source operand (gather = read + write) and the same per
    non-contiguous result operand (scatter).  Returns (copy bytes, count of copy kernels)."""
    total = 0
    kernels = 0
    for (t, members), item in zip(sched, check_ideal(m, sched, row)):
        k = len(members)
        if not item["result"]:
            total += 2 * k * row_bytes
            kernels += 1
        for ok in item["sources"]:
            if not ok:
                total += 2 * k * row_bytes
                kernels += 1
    return total, kernels
