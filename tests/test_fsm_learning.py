"""FSM learning (PAPER §2.3; §5.3): the oracle's tabular N-step Q-learning
(oracle/rl.py) pinned against what the paper and the mathematics fix, and the product learner
(ed_fsm_learn in libedbatch.so) bit-exact against the oracle.  CPU only."""
import itertools

import pytest

import workloads as W
from oracle.graph import Merged, lower_bound
from oracle.rl import RLConfig, SplitMix64, nstep_backup, policy_table, reward, train
from oracle.schedule import (agenda_chooser, depth_schedule, frontier, fsm_schedule, optimal_batches, run_alg1,
                             validate_schedule)


def instances(wl):
    return [Merged([g], len(wl.types)) for g in wl.graphs]


def trees():
    return W.treelstm(8, (2, 16), 32, "fp32", cfg=1)


# ------------------------------------------------------------------------------------------------
# oracle pins
# ------------------------------------------------------------------------------------------------

def test_splitmix64_reference_values():
    # SplitMix64 (Steele, Lea & Flood 2014; Vigna's splitmix64.c): the widely used test vector for
    # seed 1234567 (first three outputs)
    r = SplitMix64(1234567)
    assert [r.next() for _ in range(3)] == [6457827717110365317, 3203168211198807973, 9817491932198370423]


def test_reward_eq1_on_fig1_iteration2():
    """after the first I batch the ratio is 5/7 for O and 1/1 for I; Eq. 1 with alpha."""
    g, _ = W.fig1_fixture()
    m = Merged([g], 3)
    executed = [False] * m.n
    for v in frontier(m, executed):
        if m.type[v] == 0:
            executed[v] = True                      # iteration 1 batches I1
    assert reward(m, executed, 1, 0.5) == pytest.approx(-1 + 0.5 * 5 / 7)
    assert reward(m, executed, 0, 0.5) == pytest.approx(-0.5)
    assert reward(m, executed, 1, 0.0) == -1.0


def test_alpha_zero_return_is_minus_batches():
    """with alpha = 0 every step earns -1, so an episode's return is -(its batches)."""
    r = train(instances(trees()), RLConfig(alpha=0.0, max_episodes=60, check_every=1000))
    assert r.returns == [-float(b) for b in r.batches]


def test_nstep_backup_by_hand():
    """One episode of three steps, N = 2, lr = 0.5: the backup written out term by term."""
    q = {}
    trace = [((0, 1), 0, -1.0), ((1,), 1, -0.5), ((1,), 1, -0.25)]
    cfg = RLConfig(n_steps=2, lr=0.5)
    nstep_backup(q, trace, cfg)
    # t=0: G = r0 + r1 + max_b Q((1,), b) (still 0) = -1.5 -> Q = 0.5 * -1.5
    assert q[((0, 1), 0)] == -0.75
    # t=1: G = r1 + r2 (t+2 = T: no bootstrap) = -0.75 -> Q = -0.375; t=2: G = -0.25 -> Q = -0.375 - 0.5*(...)
    assert q[((1,), 1)] == pytest.approx(-0.375 + 0.5 * (-0.25 + 0.375))


def test_single_type_chain_converges_at_first_checkpoint():
    """Any policy is optimal on a single-type chain."""
    g = W.graph_from_lists([0] * 6, [[-1]] + [[k] for k in range(5)])
    m = Merged([g], 1)
    r = train([m], RLConfig(check_every=10))
    assert lower_bound(m) == 6
    assert r.checkpoints[0] == (10, 6)
    assert r.episodes == 10


def test_tree_family_reaches_lower_bound_and_batches_I_before_O():
    """the learned policy batches I while O nodes wait (O in one batch per tree), and
    reaches the App. B.3 lower bound on random parse trees."""
    ms = instances(trees())
    r = train(ms, RLConfig())
    assert r.checkpoints[-1][1] == r.lower_bound == sum(lower_bound(m) for m in ms)
    I, O = 1, 2
    for key, a in r.table.items():
        if I in key and O in key:
            assert a == I, (key, a)


def test_lattice_family_no_worse_than_depth_and_agenda():
    """Fig. 8: the FSM policy executes no more batches than the depth and agenda
    heuristics."""
    wl = W.lattice(12, (8, 16), 32, "fp32")
    ms = instances(wl)
    r = train(ms, RLConfig(max_episodes=300))
    learned = sum(len(fsm_schedule(m, r.table)) for m in ms)
    depth = sum(len(depth_schedule(m)) for m in ms)
    agenda = sum(len(run_alg1(m, agenda_chooser(m))) for m in ms)
    assert learned <= depth and learned <= agenda
    for m in ms:
        validate_schedule(m, fsm_schedule(m, r.table))


def test_two_type_family_matches_best_table_by_enumeration():
    """Brute force: with two types (BiLSTM F/B, no tagger) there are 4 E_sort tables; the learned
    table is as good as the best of them."""
    wl = W.bilstm(6, (3, 9), 32, "fp32", with_tagger=False)
    ms = instances(wl)
    r = train(ms, RLConfig(max_episodes=200))
    learned = sum(len(fsm_schedule(m, r.table)) for m in ms)
    keys = [(0, 1), (1, 0)]
    best = min(sum(len(fsm_schedule(m, {**{(0,): 0, (1,): 1}, **dict(zip(keys, ch))})) for m in ms)
               for ch in itertools.product(*keys))
    assert learned == best


def test_appendix_b4_fixture_exceeds_optimum():
    """App. B.4: the frontier-set state aliases the two halves' opposite needs, so the
    learned FSM cannot reach the optimum (found by brute force) on this fixture."""
    g, _ = W.b4_fixture()
    m = Merged([g], 3)
    opt = optimal_batches(m)
    r = train([m], RLConfig())
    assert opt == lower_bound(m)
    assert len(fsm_schedule(m, r.table)) > opt


def test_training_is_deterministic_per_seed():
    ms = instances(trees())
    a = train(ms, RLConfig(max_episodes=80, check_every=1000, seed=7))
    b = train(ms, RLConfig(max_episodes=80, check_every=1000, seed=7))
    assert a.q == b.q and a.table == b.table


# ------------------------------------------------------------------------------------------------
# product learner (C ABI) vs oracle: bit-exact tables, Q values and checkpoints
# ------------------------------------------------------------------------------------------------

CASES = [
    ("trees", lambda: trees(), dict()),
    ("trees_alpha0", lambda: trees(), dict(alpha=0.0, max_episodes=120, check_every=40)),
    ("lattice", lambda: W.lattice(10, (6, 14), 32, "fp32"), dict(max_episodes=160, check_every=40)),
    ("bilstm", lambda: W.bilstm(6, (3, 9), 32, "fp32"), dict(max_episodes=150, check_every=50, n_steps=2)),
    ("lattice_base", lambda: W.lattice(8, (6, 12), 32, "fp32"), dict(encoder="base", max_episodes=120,
                                                                      check_every=30)),
    ("treelstm_2type", lambda: W.treelstm_2type(10, (3, 14), 32, "fp32", cfg=7), dict(max_episodes=200)),
    ("lattice_max", lambda: W.lattice(8, (6, 12), 32, "fp32"), dict(encoder="max", max_episodes=120, check_every=30)),
    ("trees_max", lambda: trees(), dict(encoder="max", max_episodes=150)),
]


def _flat(key, encoder):
    """Oracle key -> C ABI key: an E_max state (set, argmax) is the set followed by the argmax type."""
    return tuple(key[0]) + (key[1],) if encoder == "max" else tuple(key)


@pytest.mark.parametrize("name,make,kw", CASES, ids=[c[0] for c in CASES])
def test_c_learner_bit_exact_with_oracle(name, make, kw):
    from paper_2302_03851_b200 import edbatch as E
    wl = make()
    cfg = RLConfig(**kw)
    ref = train(instances(wl), cfg)
    enc = {"base": E.ED_ENC_BASE, "max": E.ED_ENC_MAX}.get(cfg.encoder, E.ED_ENC_SORT)
    got = E.ed_fsm_learn(wl.graphs, wl.types, encoder=enc, alpha=cfg.alpha, lr=cfg.lr, eps0=cfg.eps0,
                         eps_decay=cfg.eps_decay, eps_every=cfg.eps_every, eps_floor=cfg.eps_floor,
                         n_steps=cfg.n_steps, max_episodes=cfg.max_episodes, check_every=cfg.check_every,
                         seed=cfg.seed)
    assert got.info["episodes"] == ref.episodes
    assert got.checkpoints == ref.checkpoints
    assert got.info["lower_bound"] == ref.lower_bound
    assert dict(got.table) == {_flat(k, cfg.encoder): a for k, a in ref.table.items()}
    assert got.q == {(_flat(k, cfg.encoder), a): v for (k, a), v in ref.q.items()}   # exact: same order
    if cfg.encoder == "max":   # the E_max table drives ed_plan exactly as the oracle's Alg. 1
        plan = E.ed_plan(wl.graphs, wl.types, got.table, encoder=E.ED_ENC_MAX)
        m = Merged(wl.graphs, len(wl.types))
        assert [(t, sorted(mem)) for t, mem in plan.schedule()] == fsm_schedule(m, ref.table, "max")


def test_learned_table_drives_ed_plan():
    """The learned table is an ed_fsm_t for ed_plan; its schedule equals the oracle's Alg. 1 run with
    the same table on the merged minibatch."""
    from paper_2302_03851_b200 import edbatch as E
    wl = trees()
    got = E.ed_fsm_learn(wl.graphs, wl.types)
    plan = E.ed_plan(wl.graphs, wl.types, got.table)
    m = Merged(wl.graphs, len(wl.types))
    ref = fsm_schedule(m, dict(got.table))
    assert [(t, sorted(mem)) for t, mem in plan.schedule()] == ref
    assert plan.info["num_batches"] == plan.info["lower_bound"]


def test_c_learner_rejects_bad_config():
    from paper_2302_03851_b200 import edbatch as E
    wl = trees()
    with pytest.raises(E.EdError) as e:
        E.ed_fsm_learn(wl.graphs, wl.types, n_steps=0)
    assert e.value.name == "ED_E_INVALID_ARG"
    with pytest.raises(E.EdError):
        E.ed_fsm_learn(wl.graphs, wl.types, lr=0.0)


def test_two_internal_types_learned_beats_priority_and_heuristics():
    """TreeLSTM-2Type (Table 1): a fixed type priority batches the two internal types apart
    and needs many more batches; the learned FSM is within a few batches of the lower bound and no
    worse than the depth / agenda heuristics (Fig. 8)."""
    from oracle.schedule import table_from_priority
    wl = W.treelstm_2type(16, (5, 20), 32, "fp32", cfg=7)
    ms = instances(wl)
    r = train(ms, RLConfig())
    learned = sum(len(fsm_schedule(m, r.table)) for m in ms)
    prio = sum(len(fsm_schedule(m, table_from_priority(wl.priority, 4))) for m in ms)
    depth = sum(len(depth_schedule(m)) for m in ms)
    agenda = sum(len(run_alg1(m, agenda_chooser(m))) for m in ms)
    assert r.lower_bound <= learned <= min(prio, depth, agenda)
    assert learned < prio


# ------------------------------------------------------------------------------------------------
# episodes over the merged minibatch (the dataflow graph ed_plan schedules)
# ------------------------------------------------------------------------------------------------

def _all_sort_tables(nt):
    """Every E_sort FSM table over nt types: one action per ordered key, chosen from the key."""
    keys = [k for r in range(1, nt + 1) for s in itertools.combinations(range(nt), r)
            for k in itertools.permutations(s)]
    for acts in itertools.product(*keys):
        yield dict(zip(keys, acts))


def test_merged_learning_matches_best_enumerated_table_on_lattice_minibatch():
    """Brute force over policies (SURVEY A-8): on a merged lattice minibatch the table learned with
    merged episodes executes as few batches as the best of all 4 E_sort tables; per-instance
    training does not see the cross-instance frontier and may not."""
    from paper_2302_03851_b200 import edbatch as E
    wl = W.lattice(96, (10, 50), 32, "fp32")
    got = E.ed_fsm_learn(wl.graphs, wl.types, merged=True)
    learned = E.ed_plan(wl.graphs, wl.types, got.table).info["num_batches"]
    best = min(E.ed_plan(wl.graphs, wl.types, list(t.items())).info["num_batches"] for t in _all_sort_tables(2))
    assert learned == best == got.info["final_batches"]
    assert got.info["lower_bound"] <= learned


@pytest.mark.parametrize("family", ["lattice", "trees"])
def test_c_learner_merged_bit_exact_with_oracle(family):
    from paper_2302_03851_b200 import edbatch as E
    wl = W.lattice(10, (6, 14), 32, "fp32") if family == "lattice" else trees()
    cfg = RLConfig(max_episodes=150, check_every=50)
    ref = train([Merged(wl.graphs, len(wl.types))], cfg)
    got = E.ed_fsm_learn(wl.graphs, wl.types, max_episodes=cfg.max_episodes, check_every=cfg.check_every,
                         merged=True)
    assert got.checkpoints == ref.checkpoints
    assert got.info["lower_bound"] == ref.lower_bound
    assert got.info["final_batches"] == ref.final_batches
    assert dict(got.table) == ref.table
    assert got.q == ref.q


def test_exported_policy_ignores_untried_actions():
    """pi(S) is the argmax over the actions with a Q entry in S; an untried action (0 by
    the exploration default) must not beat a tried one with a negative value."""
    q = {((0, 1), 1): -2.0}
    assert policy_table(q, "sort") == {(0, 1): 1}
    q[((0, 1), 0)] = -3.0
    assert policy_table(q, "sort") == {(0, 1): 1}
    q[((0, 1), 0)] = -1.0
    assert policy_table(q, "sort") == {(0, 1): 0}
