"""C-ABI tests that need no GPU: exports, ed_plan schedules/layouts vs the oracle, error codes.

ed_plan is host-only (C++), so the FSM scheduler and the layout are checked here bit-exactly
against the independent Python oracle (oracle/schedule.py, oracle/layout.py).
"""
import re
import os
import ctypes

import numpy as np
import pytest

import workloads as W
from oracle import layout as OL
from oracle import schedule as S
from oracle.graph import Merged, lower_bound_dp

E = pytest.importorskip("paper_2302_03851_b200.edbatch")

HDR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "ed_batch.h")


def test_library_exports_every_declared_symbol():
    src = open(HDR).read()
    names = set(re.findall(r"^[A-Za-z_][\w \*]*?\b(ed_\w+)\s*\(", src, flags=re.M))
    assert {"ed_plan", "ed_execute", "ed_pack_weights", "ed_plan_info", "ed_plan_destroy",
            "ed_last_error"} <= names
    for n in names:
        assert hasattr(E.LIB, n), n
    assert E.version().startswith("ed_batch")


def _plan(wl, layout=0, priority=None, encoder=0):
    pr = wl.priority if priority is None else priority
    return E.ed_plan(wl.graphs, wl.types, E.fsm_from_priority(pr, len(wl.types)), encoder=encoder, layout=layout)


def _oracle_schedule(wl, priority=None, encoder="sort"):
    m = Merged(wl.graphs, len(wl.types))
    pr = wl.priority if priority is None else priority
    return m, S.fsm_schedule(m, S.table_from_priority(pr, len(wl.types)), encoder)


def _check_schedule(wl, priority=None):
    plan = _plan(wl, priority=priority)
    m, so = _oracle_schedule(wl, priority)
    sc = plan.schedule()
    assert [(t, sorted(b)) for t, b in sc] == so
    assert plan.info["lower_bound"] == lower_bound_dp(m)
    assert plan.info["num_batches"] == len(so)
    return plan, m, so


@pytest.mark.parametrize("wlf", [
    lambda: W.config("cfg1"),
    lambda: W.treelstm(32, (1, 30), 64, "bf16", cfg=9),
    lambda: W.treelstm(20, (1, 25), 64, "fp32", cfg=10, cell="treegru"),
    lambda: W.treefc(40, (1, 30), 64, "bf16", cfg=4),
    lambda: W.treefc(40, (1, 30), 64, "bf16", cfg=4, cell="mvrnn"),
    lambda: W.bilstm(16, (1, 20), 64, "bf16", with_tagger=False),
])
def test_schedule_bit_exact_with_oracle(wlf):
    _check_schedule(wlf())


def test_schedule_bit_exact_cfg3_full_size():
    _check_schedule(W.config("cfg3"))


def test_schedule_all_priorities_tiny_trees():
    wl = W.treelstm(3, (2, 6), 32, "fp32", cfg=21)
    for pr in ([0, 1, 2], [2, 1, 0], [1, 0, 2], [0, 2, 1], [1, 2, 0], [2, 0, 1]):
        _check_schedule(wl, priority=pr)


def _fixture_types(names, h=32):
    kinds = {"I": ("treefc_internal", 2), "O": ("linear_out", 1), "R": ("treefc_internal", 2),
             "A": ("linear_out", 1), "alpha": ("treefc_internal", 2), "sigma": ("linear_out", 1)}
    return [W.OpType(n, kinds[n][0], kinds[n][1], weight_set=i, hidden=h, out_dim=4 if kinds[n][0] == "linear_out" else 0,
                     dtype="fp32") for i, n in enumerate(names)]


def test_fig1_fixture_through_the_abi():
    g, names = W.fig1_fixture()
    types = _fixture_types(names)
    plan = E.ed_plan([g], types, E.fsm_from_priority([0, 2, 1], 3))
    sc = plan.schedule()
    assert len(sc) == 10 == plan.info["lower_bound"]           # PAPER Fig. 2 / App. B.3
    assert sum(1 for t, _ in sc if t == 1) == 1                 # all O in one batch


def _random_typed_dag(rng, n):
    """Random DAG whose types have fixed arity: 0,1 -> 2 slots, 2 -> 1 slot (node or external)."""
    types, ins = [], []
    for v in range(n):
        t = rng.randint(0, 2)
        k = 2 if t < 2 else 1
        slots = []
        for _ in range(k):
            if v > 0 and rng.uniform01() < 0.8:
                slots.append(rng.randint(0, v - 1))
            else:
                slots.append(-1 - rng.randint(0, 9))
        types.append(t)
        ins.append(slots)
    return W.graph_from_lists(types, ins)


def test_random_dags_schedule_and_layout_match_oracle():
    rng = W.SplitMix64(123)
    types = [W.OpType("A", "treefc_internal", 2, weight_set=0, hidden=32, dtype="fp32"),
             W.OpType("B", "treefc_internal", 2, weight_set=1, hidden=32, dtype="fp32"),
             W.OpType("C", "linear_out", 1, weight_set=2, hidden=32, out_dim=3, dtype="fp32")]
    for trial in range(25):
        graphs = [_random_typed_dag(rng, rng.randint(1, 25)) for _ in range(rng.randint(1, 4))]
        wl = W.Workload("rand", types, graphs, [0, 1, 2], [], "fp32", 32)
        for pr in ([0, 1, 2], [2, 0, 1]):
            plan = _plan(wl, priority=pr)
            m, so = _oracle_schedule(wl, pr)
            assert [(t, sorted(b)) for t, b in plan.schedule()] == so
            row = plan.layout()
            assert list(row) == OL.schedule_order_layout(m, so)
            # CONTIG flags of the lowering == the oracle's ideal-layout check per fixed slot
            modes = plan.slot_modes()
            rep = OL.check_ideal(m, so, row)
            for b, item in enumerate(rep):
                assert item["result"]
                for j, ok in enumerate(item["sources"][:2]):
                    assert bool(modes[b, j]) == ok


def test_schedule_order_layout_results_contiguous_and_members_by_row():
    wl = W.treelstm(10, (2, 12), 32, "fp32", cfg=3)
    plan = _plan(wl)
    row = plan.layout()
    for t, mem in plan.schedule():
        rows = [row[v] for v in mem]
        assert rows == list(range(rows[0], rows[0] + len(rows)))


def test_plan_info_fields():
    wl = W.config("cfg1")
    plan = _plan(wl)
    i = plan.info
    assert i["num_nodes"] == wl.num_nodes and i["num_rows"] == wl.num_nodes + 1
    assert i["num_instances"] == len(wl.graphs) and i["hidden"] == 32 and i["dtype"] == E.ED_FP32
    assert i["workspace_bytes"] >= i["off_y"] + 4 * i["num_rows"] * i["y_cols"]
    assert i["off_h"] % 1024 == 0 and i["off_c"] % 1024 == 0
    assert i["contig_operands"] + i["gather_operands"] > 0
    assert i["plan_us"] > 0


def _expect(code, fn):
    with pytest.raises(E.EdError) as ei:
        fn()
    assert ei.value.name == code, str(ei.value)


def test_error_codes():
    t = [W.OpType("I", "treefc_internal", 2, weight_set=0, hidden=64, dtype="bf16")]
    fsm = E.fsm_from_priority([0], 1)
    cyc = W.graph_from_lists([0, 0], [[1, -1], [0, -1]])
    _expect("ED_E_CYCLE", lambda: E.ed_plan([cyc], t, fsm))
    dang = W.graph_from_lists([0], [[5, -1]])
    _expect("ED_E_DANGLING", lambda: E.ed_plan([dang], t, fsm))
    arity = W.graph_from_lists([0], [[-1]])
    _expect("ED_E_ARITY", lambda: E.ed_plan([arity], t, fsm))
    badt = W.graph_from_lists([3], [[-1, -2]])
    _expect("ED_E_TYPE", lambda: E.ed_plan([badt], t, fsm))
    ok = W.graph_from_lists([0], [[-1, -2]])
    _expect("ED_E_FSM", lambda: E.ed_plan([ok], t, [((0,), 1)]))          # action not in key
    t2 = t + [W.OpType("J", "treefc_internal", 2, weight_set=1, hidden=64, dtype="bf16")]
    _expect("ED_E_FSM", lambda: E.ed_plan([ok], t2, [((0, 0), 0)]))      # repeated type in key
    _expect("ED_E_FSM", lambda: E.ed_plan([ok], t2, [((0, 7), 0)]))      # type out of range
    odd = [W.OpType("I", "treefc_internal", 2, weight_set=0, hidden=48, dtype="bf16")]
    _expect("ED_E_TYPE", lambda: E.ed_plan([ok], odd, fsm))              # bf16 needs h % 64 == 0
    mix = [t[0], W.OpType("J", "treefc_internal", 2, weight_set=1, hidden=128, dtype="bf16")]
    _expect("ED_E_TYPE", lambda: E.ed_plan([ok], mix, E.fsm_from_priority([0, 1], 2)))


def test_null_arguments_rejected():
    out = ctypes.c_void_p()
    assert E.LIB.ed_plan(None, 1, None, 1, None, None, ctypes.byref(out)) == -1
    assert E.LIB.ed_plan_info(None, None) == -1
    assert b"bad" in E.LIB.ed_last_error() or len(E.LIB.ed_last_error()) > 0


def test_fsm_table_miss_falls_back_to_key0():
    wl = W.treelstm(6, (2, 9), 32, "fp32", cfg=5)
    plan = E.ed_plan(wl.graphs, wl.types, [])          # every lookup misses
    m = Merged(wl.graphs, 3)
    so = S.fsm_schedule(m, {})
    assert [(t, sorted(b)) for t, b in plan.schedule()] == so


def test_packed_bytes():
    h = 512
    assert E.ed_packed_bytes("treelstm_internal", h, 0, "bf16", 0) == 5 * h * 2 * h * 2
    assert E.ed_packed_bytes("treelstm_leaf", h, 0, "fp32", 0) == 3 * h * h * 4
    # bf16 output linear: UMMA layout of a zero-padded N = 16 tile; fp32: [C][h] fp32
    assert E.ed_packed_bytes("linear_out", h, 5, "bf16", 0) == 16 * h * 2
    assert E.ed_packed_bytes("linear_out", h, 5, "fp32", 0) == 5 * h * 4


def test_empty_and_degenerate_graphs():
    t = [W.OpType("I", "treefc_internal", 2, weight_set=0, hidden=64, dtype="bf16")]
    fsm = E.fsm_from_priority([0], 1)
    empty = W.Graph(np.zeros(0, np.int32), np.zeros(1, np.int32), np.zeros(0, np.int32), np.zeros(0, np.int32), -5)
    one = W.graph_from_lists([0], [[-1, -2]])
    plan = E.ed_plan([empty, one, empty], t, fsm)
    assert plan.info["num_nodes"] == 1 and plan.info["num_batches"] == 1 and plan.info["num_instances"] == 3


def test_mvrnn_plan_lowering_and_buffers():
    """MV-RNN batches lower to three device steps (matvecs, p GEMM, matrix GEMM); the workspace holds
    U [rows, 2h] and the node matrices [rows, h, h]; the word-matrix table packs to words*h*h."""
    wl = W.treefc(12, (2, 9), 64, "bf16", cfg=4, cell="mvrnn")
    plan = _plan(wl)
    i = plan.info
    assert i["num_steps"] == 3 * i["num_batches"]
    assert i["off_u"] > 0 and i["off_m"] > i["off_u"]
    rows, h = i["num_rows"], i["hidden"]
    assert i["workspace_bytes"] >= i["off_m"] + 2 * rows * h * h
    assert E.ed_packed_bytes("mvrnn_internal", 64, 100, "bf16", 2) == 100 * 64 * 64 * 2
    assert E.ed_packed_bytes("mvrnn_internal", 64, 0, "fp32", 1) == 64 * 128 * 4
    plain = _plan(W.treefc(12, (2, 9), 64, "bf16", cfg=4)).info
    assert plain["off_u"] == -1 and plain["off_m"] == -1


def test_mvrnn_rejects_bad_hidden():
    t = [W.OpType("I", "mvrnn_internal", 2, weight_set=0, hidden=4100, dtype="fp32")]
    g = W.treefc(2, (2, 4), 8, "fp32", cfg=4).graphs
    with pytest.raises(E.EdError):
        E.ed_plan(g, t, E.fsm_from_priority([0], 1))


_CODE = {v: k for k, v in E.STATUS.items()}


def _execute_host_checks(plan, sets):
    """ed_execute's host-side argument checks run before any CUDA call, so they are testable here
    with dummy (never dereferenced) pointers and a dummy 1024-aligned workspace address."""
    arr = (E.ed_weight_set_t * len(sets))(*sets)
    w = E.ed_weights_t(len(sets), arr)
    io = E.ed_io_t(None, None)
    ws = ctypes.c_void_p(1 << 40)
    return E.LIB.ed_execute(plan.handle, ctypes.byref(w), ctypes.byref(io), ws, plan.info["workspace_bytes"], None)


def _dummy_set(emb_rows=0, emb2_rows=0, W2=True):
    p = 1 << 41
    return E.ed_weight_set_t(p, p, p if W2 else None, p if W2 else None, p if emb_rows else None,
                             p if emb2_rows else None, None, emb_rows, emb2_rows)


def test_external_inputs_only_where_a_table_backs_them():
    """External ids (-1 - id) are rows of a weight set's table: TreeFC / MV-RNN children (emb) and a
    lattice word's end char (slot 1, emb2).  Elsewhere (a TreeLSTM child, a variadic word input of a
    lattice char) the kernel would index H with a negative row: the scheduler still plans the graph
    (Alg. 1 is generic), ed_execute refuses it (ED_E_UNSUPPORTED) before touching the device."""
    lstm = W.treelstm(2, (2, 4), 64, "bf16", cfg=5)
    g = lstm.graphs[0]
    bad_in = g.in_idx.copy()
    internal = [v for v in range(g.num_nodes) if lstm.types[g.type[v]].kind == "treelstm_internal"][0]
    bad_in[g.in_off[internal]] = -1 - 3
    bad = W.Graph(g.type, g.in_off, bad_in, g.ext, g.root)
    plan = E.ed_plan([bad], lstm.types, E.fsm_from_priority(lstm.priority, 3))
    sets = [_dummy_set(emb_rows=10000), _dummy_set(), _dummy_set()]
    assert _execute_host_checks(plan, sets) == _CODE["ED_E_UNSUPPORTED"]
    assert b"external" in E.LIB.ed_last_error()
    lat = W.lattice(6, (8, 14), 64, "bf16")
    for gl in lat.graphs:
        chars_with_words = [v for v in range(gl.num_nodes) if gl.type[v] == 0 and gl.in_off[v + 1] - gl.in_off[v] > 1]
        if chars_with_words:
            v = chars_with_words[0]
            li = gl.in_idx.copy()
            li[gl.in_off[v] + 1] = -1 - 2                          # variadic word slot
            badl = W.Graph(gl.type, gl.in_off, li, gl.ext, gl.root)
            p2 = E.ed_plan([badl], lat.types, E.fsm_from_priority(lat.priority, 2))
            assert _execute_host_checks(p2, [_dummy_set(4096), _dummy_set(16384, 4096)]) == _CODE["ED_E_UNSUPPORTED"]
            break
    else:
        pytest.fail("no lattice char with a word input")


def test_execute_checks_token_ids_and_weight_pointers():
    """Every token / external id a plan reads must be < the table's row count; W, b (and W2, b2 for
    the tagger and lattice word cells) must be non-null."""
    wl = W.lattice(6, (8, 14), 64, "bf16")
    plan = E.ed_plan(wl.graphs, wl.types, E.fsm_from_priority(wl.priority, 2))
    max_tok = max(int(g.ext[v]) for g in wl.graphs for v in range(g.num_nodes) if g.type[v] == 0)
    max_word = max(int(g.ext[v]) for g in wl.graphs for v in range(g.num_nodes) if g.type[v] == 1)
    ok_sets = [_dummy_set(max_tok + 1), _dummy_set(max_word + 1, 4096)]
    # all checks pass: the call gets as far as the device (none here -> a CUDA error, not a check)
    assert _execute_host_checks(plan, ok_sets) == _CODE["ED_E_CUDA"]
    assert _execute_host_checks(plan, [_dummy_set(max_tok), ok_sets[1]]) == _CODE["ED_E_INVALID_ARG"]
    assert b"emb" in E.LIB.ed_last_error()
    assert _execute_host_checks(plan, [ok_sets[0], _dummy_set(max_word)]) == _CODE["ED_E_INVALID_ARG"]
    assert _execute_host_checks(plan, [ok_sets[0], _dummy_set(max_word + 1, 4096, W2=False)]) == _CODE["ED_E_INVALID_ARG"]
    assert b"W2" in E.LIB.ed_last_error()
    # external child words of TreeFC index emb of the internal op's weight set
    fc = W.treefc(6, (2, 9), 64, "bf16", cfg=4)
    pfc = E.ed_plan(fc.graphs, fc.types, E.fsm_from_priority(fc.priority, len(fc.types)))
    max_w = max(-1 - int(x) for g in fc.graphs for x in g.in_idx if x < 0 and x != -(2 ** 31))
    assert _execute_host_checks(pfc, [_dummy_set(max_w + 1)] + [_dummy_set()] * (len(fc.types) - 1)) == _CODE["ED_E_CUDA"]
    assert _execute_host_checks(pfc, [_dummy_set(max_w)] + [_dummy_set()] * (len(fc.types) - 1)) == _CODE["ED_E_INVALID_ARG"]


@pytest.mark.parametrize("policy", ["depth", "agenda", "sc"])
def test_comparator_policies_bit_exact_with_oracle(policy):
    """The Fig. 8 comparators (P:107 depth / agenda, P:436 sufficient condition) in ed_plan equal the
    oracle's schedulers batch for batch, on the Fig. 1 fixture and on random minibatches of every
    workload family."""
    pol = {"depth": E.ED_POLICY_DEPTH, "agenda": E.ED_POLICY_AGENDA, "sc": E.ED_POLICY_SC}[policy]

    def ref(m):
        if policy == "depth":
            return S.depth_schedule(m)
        return S.run_alg1(m, S.agenda_chooser(m) if policy == "agenda" else S.sc_chooser())
    g, names = W.fig1_fixture()
    plan = E.ed_plan([g], _fixture_types(names), [], policy=pol)
    assert [(t, sorted(b)) for t, b in plan.schedule()] == ref(Merged([g], 3))
    for wl in (W.treelstm(6, (2, 9), 32, "fp32", cfg=5), W.bilstm(5, (2, 8), 32, "fp32", cfg=6),
               W.lattice(4, (3, 10), 32, "fp32", cfg=7), W.treelstm_2type(6, (2, 9), 32, "fp32", cfg=8)):
        plan = E.ed_plan(wl.graphs, wl.types, [], policy=pol)
        m = Merged(wl.graphs, len(wl.types))
        assert [(t, sorted(b)) for t, b in plan.schedule()] == ref(m), wl.name


def test_split_k_pairs_planned_for_small_tree_batches(monkeypatch):
    """Split-K over CTA pairs (reading A-28): the bf16 planner splits exactly the
    TreeLSTM / TreeGRU internal batches whose 16-unit tiles fill at most half a wave
    (2 x ceil(m / 128) x h / 16 <= 148), never the leaf or output batches, never the fp32 path,
    and not at all with ED_SPLIT=0."""
    from paper_2302_03851_b200 import edbatch as EB
    for name in ("cfg3", "cfg3_gru"):
        wl = W.config(name)
        learned = EB.ed_fsm_learn(wl.graphs, wl.types, merged=True)
        plan = EB.ed_plan(wl.graphs, wl.types, learned.table, layout=EB.ED_LAYOUT_SCHEDULE_ORDER)
        sched = plan.schedule()
        internal = [len(mem) for t, mem in sched if wl.types[t].name.startswith("I")]
        h = wl.hidden
        expect = sum(1 for m in internal if 2 * ((m + 127) // 128) * (h // 16) <= 148)
        assert expect >= 5
        assert plan.info["split_steps"] == expect, (name, internal)
    wl = W.config("cfg1")  # fp32: no tensor-core tiles, no split
    assert _plan(wl).info["split_steps"] == 0
    monkeypatch.setenv("ED_SPLIT", "0")
    wl = W.config("cfg3")
    learned = E.ed_fsm_learn(wl.graphs, wl.types, merged=True)
    assert E.ed_plan(wl.graphs, wl.types, learned.table).info["split_steps"] == 0
