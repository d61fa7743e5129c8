"""Pins for the oracle scheduler (PAPER §2, Alg. 1; App. B) — CPU only.

Each test checks the oracle against something other than itself: the paper's worked values
(tests/golden/fig1.json), closed forms, invariants (App. B.3 lower bound, Lemma 1) and brute
force on tiny graphs.
"""
import json
import os
from fractions import Fraction

import pytest

import workloads as W
from oracle import schedule as S
from oracle.graph import Merged, lower_bound, lower_bound_dp, topo_depth, typed_depth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _fig1():
    g, names = W.fig1_fixture()
    return Merged([g], 3), names, json.load(open(os.path.join(GOLD, "fig1.json")))


def test_fig1_depths_paper_values():
    m, names, gold = _fig1()
    d = topo_depth(m)
    assert sorted(d[v] for v in range(m.n) if m.type[v] == 0) == gold["I_depths"]
    assert sorted(d[v] for v in range(m.n) if m.type[v] == 1) == gold["O_depths"]
    o = [d[v] for v in range(m.n) if m.type[v] == 1]
    i = [d[v] for v in range(m.n) if m.type[v] == 0]
    assert Fraction(sum(o), len(o)) == Fraction(*gold["O_mean_depth"])      # 13/7 = 1.857
    assert Fraction(sum(i), len(i)) == Fraction(*gold["I_mean_depth"])      # 2


def test_fig1_depth_based_runs_O_in_four_batches():
    m, names, gold = _fig1()
    s = S.depth_schedule(m)
    S.validate_schedule(m, s)
    assert sum(1 for t, _ in s if t == 1) == gold["depth_based_O_batches"]
    assert len(s) == 13                                                       # SPEC S:180 (derived)


def test_fig1_agenda_picks_O_after_first_I_batch():
    m, names, gold = _fig1()
    executed = [False] * m.n
    executed[0] = True  # the first I batch (I1)
    front = S.frontier(m, executed)
    counts = S.type_counts(m, front)
    pick = S.agenda_chooser(m)(m, executed, front, counts)
    assert names[pick] == gold["agenda_pick_after_first_I"]


def test_fig1_fsm_policy_batches_all_O_once_and_hits_lower_bound():
    m, names, gold = _fig1()
    # Fig. 2 policy: {I,O}->I, {O}->O, {O,R}->R, {R}->R  == priority I > R > O on E_sort keys
    table = S.table_from_priority([0, 2, 1], 3)
    for key_s, act in gold["fsm_fig2_policy"].items():
        ts = [names.index(x) for x in key_s.split(",")]
        for key in table:
            if sorted(key) == sorted(ts):
                assert names[table[key]] == act
    s = S.fsm_schedule(m, table)
    S.validate_schedule(m, s)
    assert sum(1 for t, _ in s if t == 1) == gold["fsm_O_batches"]
    assert len(s) == lower_bound(m) == 10
    assert S.optimal_batches(m) == 10


def test_fig1_eq1_ratios_at_iteration_2():
    m, names, gold = _fig1()
    executed = [False] * m.n
    executed[0] = True
    assert Fraction(S.readiness_ratio(m, executed, 1)).limit_denominator(100) == Fraction(*gold["ratio_iter2"]["O"])
    assert S.readiness_ratio(m, executed, 0) == 1.0
    # the sufficient-condition heuristic therefore keeps batching I
    front = S.frontier(m, executed)
    assert S.sc_chooser()(m, executed, front, S.type_counts(m, front)) == 0


def test_esort_encoding_order_and_ties():
    assert S.e_sort({0: 1, 1: 5}) == (1, 0)
    assert S.e_sort({0: 2, 1: 2}) == (0, 1)
    assert S.e_base({2: 1, 0: 3}) == (0, 2)
    assert S.e_max({0: 2, 1: 2}) == ((0, 1), 0)


def test_fsm_fallback_is_first_key_element():
    g = W.graph_from_lists([0, 1, 1], [[], [], []])
    m = Merged([g], 2)
    s = S.fsm_schedule(m, {})            # empty table: every state misses
    assert [t for t, _ in s] == [1, 0]   # key (1, 0): type 1 has 2 ready nodes


def _random_dag(rng, n, ntypes, pedge=0.3):
    types, ins = [], []
    for v in range(n):
        types.append(rng.randint(0, ntypes - 1))
        ins.append([u for u in range(v) if rng.uniform01() < pedge])
    return W.graph_from_lists(types, ins)


def test_lower_bound_definition_vs_dp_and_schedules():
    rng = W.SplitMix64(77)
    for _ in range(60):
        g = _random_dag(rng, rng.randint(1, 14), 3)
        m = Merged([g], 3)
        lb = lower_bound(m)
        assert lb == lower_bound_dp(m)
        for sched in (S.depth_schedule(m), S.run_alg1(m, S.agenda_chooser(m)),
                      S.run_alg1(m, S.sc_chooser()),
                      S.fsm_schedule(m, S.table_from_priority([0, 1, 2], 3))):
            assert S.validate_schedule(m, sched) >= lb                       # App. B.3
        assert S.optimal_batches(m) >= lb


def test_lemma1_sufficient_condition_brute_force():
    """App. B.2: ratio(a) = 1 at the initial state => a shortest sequence starts with a."""
    rng = W.SplitMix64(5)
    checked = 0
    for _ in range(220):
        g = _random_dag(rng, rng.randint(2, 12), 3, 0.25)
        m = Merged([g], 3)
        ex = [False] * m.n
        opt = S.optimal_batches(m)
        for a in sorted(set(m.type[v] for v in S.frontier(m, ex))):
            if S.readiness_ratio(m, ex, a) == 1.0:
                assert S.optimal_batches(m, first=a) == opt
                checked += 1
    assert checked > 100


def test_single_type_chain_closed_form():
    for n in (1, 2, 7):
        g = W.graph_from_lists([0] * n, [[]] + [[v - 1] for v in range(1, n)])
        m = Merged([g], 1)
        assert len(S.fsm_schedule(m, S.table_from_priority([0], 1))) == n == lower_bound(m)


def test_bilstm_chain_closed_form_2maxlen_plus_1():
    wl = W.bilstm(6, (3, 7), 8, "fp32", cfg=2)
    m = Merged(wl.graphs, 3)
    s = S.fsm_schedule(m, S.table_from_priority(wl.priority, 3))
    maxlen = max((g.num_nodes // 3) for g in wl.graphs)
    assert len(s) == 2 * maxlen + 1 == lower_bound(m)


def test_tiny_trees_fsm_equals_optimum_equals_lb():
    for seed in range(30):
        wl = W.treelstm(2, (2, 5), 4, "fp32", cfg=100 + seed)
        m = Merged(wl.graphs, 3)
        s = S.fsm_schedule(m, S.table_from_priority([0, 1, 2], 3))
        S.validate_schedule(m, s)
        assert len(s) == lower_bound(m) == S.optimal_batches(m)


def test_tiny_trees_fixed_table_is_best_of_all_tables():
    """BJ "batch counts match brute-force optimal policies": enumerate every E_sort table."""
    wl = W.treelstm(2, (3, 4), 4, "fp32", cfg=7)
    m = Merged(wl.graphs, 3)
    fixed = len(S.fsm_schedule(m, S.table_from_priority([0, 1, 2], 3)))
    best = min(len(S.fsm_schedule(m, t)) for t in S.enumerate_sort_tables(3))
    assert fixed == best == S.optimal_batches(m)


def test_enumerate_tables_counts():
    assert sum(1 for _ in S.enumerate_sort_tables(2)) == 4
    assert sum(1 for _ in S.enumerate_sort_tables(3)) == 46656


def test_lattice_schedules_valid_and_above_lb():
    wl = W.lattice(4, (4, 9), 4, "fp32", cfg=5)
    m = Merged(wl.graphs, 2)
    for pr in ([0, 1], [1, 0]):
        s = S.fsm_schedule(m, S.table_from_priority(pr, 2))
        assert S.validate_schedule(m, s) >= lower_bound(m)


def test_validator_rejects_bad_schedules():
    g = W.graph_from_lists([0, 0, 1], [[], [0], [1]])
    m = Merged([g], 2)
    with pytest.raises(AssertionError):
        S.validate_schedule(m, [(0, [0, 1]), (1, [2])])   # 1 depends on 0 in the same batch
    with pytest.raises(AssertionError):
        S.validate_schedule(m, [(0, [0]), (0, [1])])       # node 2 missing
    with pytest.raises(AssertionError):
        S.validate_schedule(m, [(0, [0]), (1, [1]), (1, [2])])  # wrong type
