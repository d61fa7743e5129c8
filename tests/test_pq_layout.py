"""PQ-tree layout planner (PAPER §3.2, Alg. 2-6, App. C): oracle pins and C++ bit-exactness.

Pins of the oracle (oracle/pqtree.py) against things other than itself:
  * Reduce: the tree's frontier equals, by brute force over all permutations (n <= 8), the set of
    orders keeping every accepted constraint consecutive; a Reduce fails iff that set is empty.
  * Fig. 3 (tests/golden/fig3.json): the paper's zero-copy order, and the label order's
    2 gathers + 1 scatter.
  * Chains: every constrained chain operand becomes contiguous (a zero-copy layout exists).
  * Plain definition: every batch the planner keeps satisfies adjacency + alignment (check_ideal).
Then the C++ planner (ED_LAYOUT_PQ through ed_plan) must equal the oracle layout bit for bit.
"""
import itertools
import json
import os

import numpy as np
import pytest

import workloads as W
from oracle import layout as OL
from oracle import schedule as S
from oracle.graph import Merged
from oracle.pqtree import Fail, PQTree, plan_pq_layout

E = pytest.importorskip("paper_2302_03851_b200.edbatch")
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _consecutive(perm, cons):
    pos = {v: i for i, v in enumerate(perm)}
    for c in cons:
        p = sorted(pos[v] for v in c)
        if p[-1] - p[0] != len(p) - 1:
            return False
    return True


def test_reduce_frontier_equals_brute_force():
    rng = W.SplitMix64(99)
    cases = 0
    for _ in range(400):
        n = rng.randint(2, 6)
        T = PQTree(range(n))
        accepted = []
        for _ in range(rng.randint(1, 5)):
            k = rng.randint(2, n)
            c = set()
            while len(c) < k:
                c.add(rng.randint(0, n - 1))
            c = frozenset(c)
            brute = {p for p in itertools.permutations(range(n)) if _consecutive(p, accepted + [c])}
            import copy
            saved = copy.deepcopy(T.root)
            try:
                T.reduce(c)
                ok = True
            except Fail:
                ok = False
                T.root = saved
            assert ok == bool(brute), (n, accepted, c)
            if ok:
                accepted.append(c)
                assert T.all_frontiers() == brute
            cases += 1
    assert cases > 500


def test_reduce_frontier_equals_brute_force_n7_n8():
    """The same pin at n = 7 and 8 (SURVEY O-4 "n <= 8"): the brute-force set of admissible
    orders is kept as an array of all n! permutations, filtered constraint by constraint."""
    import copy
    rng = W.SplitMix64(2024)
    cases = 0
    for n in (7, 8):
        perms = np.array(list(itertools.permutations(range(n))), dtype=np.int8)
        pos = np.argsort(perms, axis=1)                     # pos[p, v] = position of v in perm p
        for _ in range(30):
            T = PQTree(range(n))
            alive = np.ones(len(perms), dtype=bool)
            for _ in range(rng.randint(1, 7)):
                k = rng.randint(2, n - 1)
                c = set()
                while len(c) < k:
                    c.add(rng.randint(0, n - 1))
                pc = pos[:, sorted(c)]
                keep = alive & (pc.max(axis=1) - pc.min(axis=1) == len(c) - 1)
                saved = copy.deepcopy(T.root)
                try:
                    T.reduce(frozenset(c))
                    ok = True
                except Fail:
                    ok = False
                    T.root = saved
                assert ok == bool(keep.any()), (n, sorted(c))
                if ok:
                    alive = keep
                    assert T.all_frontiers() == {tuple(int(x) for x in p) for p in perms[alive]}
                cases += 1
    assert cases > 100


def _random_dag(rng, n):
    """Random DAG, types 0, 1 with two slots and 2 with one (node inputs, else external)."""
    types, ins = [], []
    for v in range(n):
        t = rng.randint(0, 2)
        slots = [rng.randint(0, v - 1) if v > 0 and rng.uniform01() < 0.85 else -1 - rng.randint(0, 9)
                 for _ in range(2 if t < 2 else 1)]
        types.append(t)
        ins.append(slots)
    return W.graph_from_lists(types, ins)


def _c1p_pass1_brute(n, ops):
    """The transactional source pass (A-9) written as the mathematical fact it implements, with no
    PQ tree: a batch is accepted iff (every result set, every set accepted so far, and all of this
    batch's source sets) are simultaneously consecutive in some order of the n variables."""
    perms = np.array(list(itertools.permutations(range(n))), dtype=np.int8)
    pos = np.argsort(perms, axis=1)

    def consecutive(alive, c):
        pc = pos[:, sorted(c)]
        return alive & (pc.max(axis=1) - pc.min(axis=1) == len(c) - 1)
    alive = np.ones(len(perms), dtype=bool)
    for o in ops:
        alive = consecutive(alive, o[0])
    acc = []
    for o in ops:
        if len(o) < 2:
            acc.append(True)
            continue
        cand = alive
        for S_ in o[1:]:
            cand = consecutive(cand, S_)
        acc.append(bool(cand.any()))
        if cand.any():
            alive = cand
    return acc


def test_source_pass_accepts_exactly_the_c1p_batches():
    """SURVEY O-4: accept / reject of each batch's source constraints is "is the accepted set union
    this batch's sets C1P?", checked here by brute force over all orders of <= 8 variables on random
    tiny minibatches (TreeFC forests, BiLSTM chains, lattices), independently of the PQ tree."""
    from oracle.pqtree import batch_operands
    types = [W.OpType("A", "treefc_internal", 2, weight_set=0, hidden=32, dtype="fp32"),
             W.OpType("B", "treefc_internal", 2, weight_set=1, hidden=32, dtype="fp32"),
             W.OpType("C", "linear_out", 1, weight_set=2, hidden=32, out_dim=3, dtype="fp32")]
    rng = W.SplitMix64(77)
    checked = rejected = 0
    for seed in range(240):
        kind = seed % 4
        if kind == 0:
            wl = W.treefc(W.SplitMix64(seed).randint(2, 4), (2, 4), 32, "fp32", cfg=3000 + seed)
        elif kind == 1:
            wl = W.bilstm(W.SplitMix64(seed).randint(2, 3), (1, 3), 32, "fp32", cfg=3000 + seed, with_tagger=False)
        elif kind == 2:
            wl = W.lattice(2, (2, 4), 32, "fp32", cfg=3000 + seed)
        else:   # random typed DAGs: two-slot ops reading shared inputs in conflicting orders
            graphs = [_random_dag(rng, rng.randint(3, 8 - 2 * k)) for k in range(rng.randint(1, 2))]
            wl = W.Workload("rand", types, graphs, [0, 1, 2], [], "fp32", 32)
        m = Merged(wl.graphs, len(wl.types))
        if not 2 <= m.n <= 8:
            continue
        sched = S.fsm_schedule(m, S.table_from_priority(wl.priority, len(wl.types)))
        fixed = [t.num_slots for t in wl.types]
        tr = {}
        plan_pq_layout(m, sched, fixed, trace=tr)
        assert tr["pass1"] == _c1p_pass1_brute(m.n, batch_operands(m, sched, fixed)), seed
        checked += 1
        rejected += tr["pass1"].count(False)
    assert checked >= 60 and rejected > 0, (checked, rejected)


def _fig3_types():
    return [W.OpType("A", "linear_out", 1, weight_set=0, hidden=32, out_dim=4, dtype="fp32"),
            W.OpType("alpha", "treefc_internal", 2, weight_set=1, hidden=32, dtype="fp32"),
            W.OpType("sigma", "linear_out", 1, weight_set=2, hidden=32, out_dim=4, dtype="fp32")]


def test_fig3_paper_layout_oracle_and_cpp():
    gold = json.load(open(os.path.join(GOLD, "fig3.json")))
    g, names = W.fig3_fixture()
    m = Merged([g], 3)
    sched = S.fsm_schedule(m, S.table_from_priority([0, 1, 2], 3))
    row, alive = plan_pq_layout(m, sched, [1, 2, 1])
    order = ["x%d" % (v + 1) for v in np.argsort(row)]
    assert order == gold["zero_copy_order"]
    assert all(alive)
    assert OL.paper_copy_kernels(m, sched, row) == (0, 0)
    label = list(range(8))
    g_, s_ = OL.paper_copy_kernels(m, sched, label)
    # label order needs 2 gathers + 1 scatter = 3 copy kernels.  The fewest-copies member
    # order gives the total; the paper's split itself follows from its batched program, Fig. 3(b),
    # whose members are listed in their first source operand's order (reading A-25b):
    assert g_ + s_ == gold["label_order_copies"]["gathers"] + gold["label_order_copies"]["scatters"]
    assert OL.executor_copy_split(m, sched, label) == (gold["label_order_copies"]["gathers"],
                                                        gold["label_order_copies"]["scatters"])
    assert OL.executor_copy_split(m, sched, row) == (0, 0)
    plan = E.ed_plan([g], _fig3_types(), E.fsm_from_priority([0, 1, 2], 3), layout=E.ED_LAYOUT_PQ)
    assert list(plan.layout()) == row
    assert plan.slot_modes()[1].tolist() == [1, 1] and plan.slot_modes()[2][0] == 1


def _both(wl, priority=None):
    pr = wl.priority if priority is None else priority
    plan = E.ed_plan(wl.graphs, wl.types, E.fsm_from_priority(pr, len(wl.types)), layout=E.ED_LAYOUT_PQ)
    m = Merged(wl.graphs, len(wl.types))
    so = S.fsm_schedule(m, S.table_from_priority(pr, len(wl.types)))
    row, alive = plan_pq_layout(m, so, [t.num_slots for t in wl.types])
    return plan, m, so, row, alive


@pytest.mark.parametrize("wlf", [
    lambda s: W.treelstm(4, (1, 12), 64, "bf16", cfg=500 + s),
    lambda s: W.treelstm(3, (1, 10), 64, "bf16", cfg=600 + s, cell="treegru"),
    lambda s: W.treefc(6, (1, 12), 64, "bf16", cfg=700 + s),
    lambda s: W.bilstm(4, (1, 9), 64, "bf16", cfg=800 + s),
    lambda s: W.lattice(3, (1, 12), 64, "fp32", cfg=900 + s),
    lambda s: W.lattice(3, (1, 12), 64, "fp32", cfg=950 + s, priority=(1, 0)),
])
def test_cpp_pq_layout_bit_exact_with_oracle(wlf):
    for s in range(25):
        plan, m, so, row, alive = _both(wlf(s))
        assert list(plan.layout()) == row
        rep = OL.check_ideal(m, so, row)
        for (t, mem), item, ok in zip(so, rep, alive):
            assert item["result"]                                            # results contiguous (A-9)
            if ok and len(mem) > 1:
                fixed = [j for j in range(m.num_types and 2)]
                # every constrained source of a kept batch is adjacent and aligned
                mm = sorted(mem)
                for j, good in enumerate(item["sources"]):
                    ent = [m.inputs[v][j] for v in mm]
                    constrained = all(k == "n" for k, _ in ent) and len({u for _, u in ent}) == len(ent)
                    if constrained and j < [tp.num_slots for tp in wlf(s).types][t]:
                        assert good, (t, j)


def test_cpp_pq_random_typed_dags_bit_exact():
    rng = W.SplitMix64(321)
    types = [W.OpType("A", "treefc_internal", 2, weight_set=0, hidden=64, dtype="bf16"),
             W.OpType("B", "treefc_internal", 2, weight_set=1, hidden=64, dtype="bf16"),
             W.OpType("C", "linear_out", 1, weight_set=2, hidden=64, out_dim=3, dtype="bf16")]
    for _ in range(60):
        graphs = []
        for _ in range(rng.randint(1, 3)):
            n = rng.randint(1, 14)
            tys, ins = [], []
            for v in range(n):
                t = rng.randint(0, 2)
                k = 2 if t < 2 else 1
                ins.append([rng.randint(0, v - 1) if v > 0 and rng.uniform01() < 0.85 else -1 - rng.randint(0, 5)
                            for _ in range(k)])
                tys.append(t)
            graphs.append(W.graph_from_lists(tys, ins))
        wl = W.Workload("rand", types, graphs, [0, 1, 2], [], "bf16", 64)
        plan, m, so, row, alive = _both(wl)
        assert list(plan.layout()) == row


def test_chains_become_fully_contiguous():
    """Single-direction chains: a zero-copy layout exists; the planner finds it."""
    wl = W.bilstm(12, (1, 20), 64, "bf16", cfg=77, with_tagger=False)
    plan, m, so, row, alive = _both(wl)
    modes = plan.slot_modes()
    for b, (t, mem) in enumerate(so):
        ent = [m.inputs[v][0] for v in mem]
        if all(k == "n" for k, _ in ent):
            assert modes[b, 0] == 1, b


def test_pq_improves_contiguity_over_schedule_order():
    """The PQ planner's objective (operands made contiguous) is at least what the schedule-order
    layout reaches.  Since reading L-3 orders each batch by its members' consumers, the schedule-order
    layout already makes single-direction chains contiguous (BiLSTM: equal); lattices still gain."""
    for wl, strict in ((W.bilstm(16, (1, 30), 64, "bf16", cfg=2), False), (W.lattice(16, (2, 30), 64, "bf16", cfg=5), True)):
        pr = E.fsm_from_priority(wl.priority, len(wl.types))
        a = E.ed_plan(wl.graphs, wl.types, pr, layout=E.ED_LAYOUT_SCHEDULE_ORDER).info
        b = E.ed_plan(wl.graphs, wl.types, pr, layout=E.ED_LAYOUT_PQ).info
        assert b["contig_operands"] >= a["contig_operands"] and b["copy_bytes"] <= a["copy_bytes"]
        if strict:
            assert b["contig_operands"] > a["contig_operands"]


@pytest.mark.parametrize("wlf", [
    lambda: W.treelstm(12, (2, 12), 32, "fp32", cfg=5),
    lambda: W.bilstm(8, (2, 12), 32, "fp32", cfg=6),
    lambda: W.lattice(6, (4, 12), 32, "fp32", cfg=7),
    lambda: W.treefc(12, (2, 12), 32, "fp32", cfg=8),
])
def test_pq_layout_avoids_copies_of_the_label_layout(wlf):
    """P:158 and Table 4: allocating memory by the PQ tree instead of by variable label
    removes gather / scatter copies.  Copy bytes and copy kernels (oracle.layout.copy_bytes, a
    DyNet-style executor) of the PQ layout against the label (node id) layout, and PQ needs no
    more copy kernels than the schedule-order layout (L-1)."""
    wl = wlf()
    m = Merged(wl.graphs, len(wl.types))
    so = S.fsm_schedule(m, S.table_from_priority(wl.priority, len(wl.types)))
    row, _ = plan_pq_layout(m, so, [t.num_slots for t in wl.types])
    pq_bytes, pq_kernels = OL.copy_bytes(m, so, row, 64)
    label_bytes, label_kernels = OL.copy_bytes(m, so, list(range(m.n)), 64)
    _, sched_kernels = OL.copy_bytes(m, so, OL.schedule_order_layout(m, so), 64)
    assert pq_bytes < label_bytes and pq_kernels < label_kernels
    assert pq_kernels <= sched_kernels


def test_static_subgraph_ablation_pq_leaves_only_broadcasts():
    """Table 4 / P:438: on the cells' static subgraphs the PQ layout removes every gather / scatter
    except broadcasts (x read by every gate) -- the "ideal memory allocation order" -- and needs far
    fewer copy kernels and bytes than the label layout.  Reading S-2 decompositions (script)."""
    import importlib.util
    path = os.path.join(os.path.dirname(os.path.dirname(__file__)), "scripts", "static_subgraph_ablation.py")
    spec = importlib.util.spec_from_file_location("ssa", path)
    ssa = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(ssa)
    types = [W.OpType(k, ssa.KINDS[k][0], ssa.KINDS[k][1], weight_set=i, hidden=ssa.H,
                      has_ext=1 if ssa.KINDS[k][1] == 0 else 0, out_dim=1 if ssa.KINDS[k][0] == "linear_out" else 0,
                      dtype="fp32") for i, k in enumerate(ssa.ORDER)]
    for name in ("LSTMCell", "GRUCell", "TreeLSTM-Internal", "TreeLSTM-Leaf", "TreeGRU-Leaf"):
        s = ssa.build(name)
        ext = [v if ssa.KINDS[s.kind[v]][1] == 0 else -1 for v in range(len(s.kind))]
        g = W.graph_from_lists([ssa.ORDER.index(k) for k in s.kind], s.ins, ext, root=len(s.kind) - 1)
        pq = E.ed_plan([g], types, [], policy=E.ED_POLICY_AGENDA, layout=E.ED_LAYOUT_PQ)
        sched = pq.schedule()
        k_label, b_label = ssa.copies(sched, list(range(len(s.kind))), s)
        k_pq, b_pq = ssa.copies(sched, list(pq.layout()), s)
        k_bc, b_bc = ssa.copies(sched, list(pq.layout()), s, broadcasts_only=True)
        assert (k_pq, b_pq) == (k_bc, b_bc), name          # only broadcasts remain
        assert k_pq < k_label and 20 * b_pq < b_label, name
