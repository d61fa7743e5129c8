"""GPU parity: the CUDA path (through the C ABI) vs the fp64 oracle, element by element.

Tolerances (BASELINE.json north_star; metric = DESIGN.md reading A-19): max relative error
<= 1e-4 for the fp32 path and <= 2e-2 for the bf16 path, per output tensor (h, c, logits, roots).
Sizes span several 128-row tiles with a ragged tail; the BASELINE full size (cfg3) is checked on
a sampled set of instances in the exact launch configuration bench.py times.
"""
import numpy as np
import pytest
import torch

import workloads as W
from harness import TOL, compare, run_gpu

pytestmark = pytest.mark.gpu


def _check(wl, instances=None, layout=0):
    plan, w, ws, out = run_gpu(wl, layout=layout)
    err = compare(wl, plan, ws, out, instances)
    tol = TOL[wl.dtype]
    assert all(v <= tol for v in err.values()), err
    return plan, w, ws, out, err


def test_cfg1_treelstm_h32_fp32_all_nodes():
    _check(W.config("cfg1"))


@pytest.mark.parametrize("h", [64, 128, 256])
def test_treelstm_bf16_ragged_tiles(h):
    # ~40 trees -> batches of 1..~600 rows: several tiles plus ragged tails and m = 1 steps
    _check(W.treelstm(40, (1, 30), h, "bf16", cfg=30 + h))


def test_treelstm_fp32_h64():
    _check(W.treelstm(24, (1, 20), 64, "fp32", cfg=31))


def test_cfg3_full_size_sampled_instances():
    wl = W.config("cfg3")
    sizes = [g.num_nodes for g in wl.graphs]
    tallest = list(np.argsort(sizes)[-8:])
    rng = np.random.default_rng(7)
    rest = list(rng.choice(len(wl.graphs), 24, replace=False))
    _check(wl, sorted(set(int(x) for x in tallest + rest)))


@pytest.mark.parametrize("dtype,h", [("bf16", 128), ("fp32", 64)])
def test_treegru(dtype, h):
    _check(W.treelstm(24, (1, 24), h, dtype, cfg=40, cell="treegru"))


@pytest.mark.parametrize("dtype,h", [("bf16", 128), ("fp32", 64)])
def test_treefc_with_external_leaves_and_single_leaf_instances(dtype, h):
    wl = W.treefc(30, (1, 24), h, dtype, cfg=41)
    # a 1-leaf instance has no ops; its output is the external (word) row itself
    wl.graphs.insert(3, W.Graph(np.zeros(0, np.int32), np.zeros(1, np.int32), np.zeros(0, np.int32),
                                np.zeros(0, np.int32), -1 - 17))
    _check(wl)


@pytest.mark.parametrize("dtype,h", [("bf16", 64), ("bf16", 128), ("bf16", 192), ("fp32", 32)])
def test_mvrnn(dtype, h):
    """MV-RNN: p (h), node matrices P (compared transposed back), roots.  h = 64: a 128-row tile of
    the matrix product spans two nodes; h = 192: tiles straddle node blocks at 64-row granularity."""
    wl = W.treefc(10, (1, 12), h, dtype, cfg=45, cell="mvrnn")
    plan, w, ws, out, err = _check(wl)
    assert "M" in err and "h" in err


def test_cfg4_mvrnn_full_size_sampled():
    """BASELINE cfg4 MV-RNN (1024 trees, h = 512, bf16) in bench.py's launch configuration; the oracle
    evaluates sampled instances (4h^3 = 537 MFLOP per node in fp64)."""
    wl = W.config("cfg4_mvrnn")
    _check(wl, list(range(0, 1024, 97)))


@pytest.mark.parametrize("dtype,h", [("bf16", 128), ("fp32", 64)])
def test_bilstm_chains(dtype, h):
    _check(W.bilstm(20, (1, 30), h, dtype, cfg=42, with_tagger=False))


@pytest.mark.parametrize("dtype,h", [("bf16", 256), ("fp32", 64)])
def test_bilstm_tagger(dtype, h):
    _check(W.bilstm(16, (1, 30), h, dtype, cfg=47))


def test_cfg2_full_size():
    _check(W.config("cfg2"))


@pytest.mark.parametrize("dtype,h", [("bf16", 128), ("fp32", 64)])
@pytest.mark.parametrize("priority", [[0, 1], [1, 0]])
def test_lattice(dtype, h, priority):
    wl = W.lattice(24, (1, 40), h, dtype, cfg=48, priority=priority)
    _check(wl)


def test_cfg5_full_size_sampled():
    wl = W.config("cfg5")
    _check(wl, list(range(0, 512, 9)))


def test_single_node_and_single_leaf_trees():
    wl = W.treelstm(9, (1, 1), 64, "bf16", cfg=43)   # every instance: one leaf + its O
    _check(wl)


def test_repeat_execute_is_bitwise_deterministic():
    from paper_2302_03851_b200 import edbatch as E
    wl = W.treelstm(30, (2, 25), 128, "bf16", cfg=44)
    plan, w, ws, out = run_gpu(wl)
    h1 = ws.H().clone(); c1 = ws.C().clone(); y1 = ws.Y().clone()
    E.ed_execute(plan, w, ws, out)
    torch.cuda.synchronize()
    assert torch.equal(h1, ws.H()) and torch.equal(c1, ws.C()) and torch.equal(y1, ws.Y())


def test_step_timestamps_cover_every_batch():
    wl = W.treelstm(16, (2, 16), 64, "bf16", cfg=45)
    plan, w, ws, out = run_gpu(wl)
    dt = ws.step_times_ns()
    assert len(dt) == plan.info["num_batches"] and np.all(dt > 0)


def test_workspace_too_small_is_rejected():
    from paper_2302_03851_b200 import edbatch as E
    wl = W.treelstm(4, (2, 5), 64, "bf16", cfg=46)
    plan, w, ws, out = run_gpu(wl)
    ws.nbytes = plan.info["workspace_bytes"] - 1024
    with pytest.raises(E.EdError) as ei:
        E.ed_execute(plan, w, ws, out)
    assert ei.value.name == "ED_E_WORKSPACE"


# ---- PQ-tree layout (ED_LAYOUT_PQ): parity, CONTIG (TMA box) operands, bitwise layout invariance ----

def _node_records(plan, ws):
    """Per global node id: (h row, c row, y row) read through the plan's layout."""
    row = plan.layout()
    H, C, Y = ws.H().float().cpu().numpy(), ws.C().cpu().numpy(), ws.Y().cpu().numpy()
    return H[row], C[row], Y[row] if Y.size else None


@pytest.mark.parametrize("wlf", [
    lambda: W.bilstm(24, (1, 40), 128, "bf16", cfg=60),
    lambda: W.bilstm(12, (1, 20), 64, "fp32", cfg=61),
    lambda: W.lattice(32, (1, 40), 128, "bf16", cfg=62),
    lambda: W.treelstm(40, (1, 30), 128, "bf16", cfg=63),
])
def test_pq_layout_parity_and_bitwise_layout_invariance(wlf):
    wl = wlf()
    plan_pq, _, ws_pq, out_pq, _ = _check(wl, layout=1)
    assert plan_pq.info["contig_operands"] > 0
    plan_s, _, ws_s, out_s = run_gpu(wl, layout=0)
    a = _node_records(plan_pq, ws_pq)
    b = _node_records(plan_s, ws_s)
    for x, y in zip(a, b):
        if x is not None:
            assert np.array_equal(x, y)          # same bits whatever row a node lives in
    assert torch.equal(out_pq, out_s)


def test_cfg2_pq_layout_full_size():
    _check(W.config("cfg2"), layout=1)


@pytest.mark.parametrize("wlf", [
    lambda: W.treelstm(60, (1, 40), 128, "bf16", cfg=65),
    lambda: W.lattice(160, (1, 30), 128, "bf16", cfg=66),
    lambda: W.bilstm(150, (1, 12), 64, "bf16", cfg=67),
])
def test_staged_operands_are_bitwise_invisible(wlf):
    """Staging (S-1) only changes where the loaders read an operand from: every node record
    and root is bit-identical with and without it (and matches the oracle)."""
    wl = wlf()
    plan_a, _, ws_a, out_a, _ = _check(wl)
    assert plan_a.info["staged_operands"] > 0
    plan_b, _, ws_b, out_b = run_gpu(wl, staging=1)
    assert plan_b.info["staged_operands"] == 0
    for x, y in zip(_node_records(plan_a, ws_a), _node_records(plan_b, ws_b)):
        if x is not None:
            assert np.array_equal(x, y)
    assert torch.equal(out_a, out_b)


def test_treelstm_2type_with_learned_fsm():
    """TreeLSTM-2Type (Table 1) planned with the Q-learned FSM (paper §2.3): two internal types
    with separate weight sets in one persistent launch; parity with the oracle."""
    from paper_2302_03851_b200 import edbatch as E
    wl = W.treelstm_2type(48, (1, 30), 128, "bf16", cfg=68)
    learned = E.ed_fsm_learn(wl.graphs, wl.types)
    plan, w, ws, out = run_gpu(wl, fsm=learned.table)
    err = compare(wl, plan, ws, out)
    assert all(v <= TOL[wl.dtype] for v in err.values()), err
    prio = E.ed_plan(wl.graphs, wl.types, E.fsm_from_priority(wl.priority, len(wl.types)))
    assert plan.info["num_batches"] <= prio.info["num_batches"]


@pytest.mark.parametrize("dtype,h", [("bf16", 128), ("fp32", 64)])
def test_latticegru(dtype, h):
    """LatticeGRU (A-27): GRU char cells max-pooled with word GRU states."""
    _check(W.lattice(40, (1, 40), h, dtype, cfg=49, cell="latticegru"))


def test_cfg5_latticegru_full_size_sampled():
    wl = W.config("cfg5_gru")
    _check(wl, list(range(0, 512, 37)))


@pytest.mark.parametrize("h", [192, 128])
def test_small_contiguous_tiles_with_single_chunk_last_stage(h):
    """Regression: a small tile (several K chunks per stage) whose last stage holds one chunk of a
    contiguous operand must gather it, not load a 128-row TMA box over the stage's B region
    (h = 192: 6 K chunks = stages of 5 + 1 for 8-row tiles)."""
    _check(W.bilstm(8, (6, 14), h, "bf16", cfg=71, with_tagger=False))


def test_repeated_launches_rebinding_and_two_workspaces():
    """Readiness counters are monotonic over launches (no per-launch memset): many executes of one
    plan, a second workspace bound in between, and a released + rebound workspace all give the
    bitwise-same node records and instance outputs as the first launch."""
    from paper_2302_03851_b200 import edbatch as E
    wl = W.treelstm(40, (1, 30), 128, "bf16", cfg=72)
    plan, w, ws, out = run_gpu(wl)
    ref_h, ref_out = ws.H().clone(), out.clone()
    ws2 = E.Workspace(plan)
    out2 = torch.zeros_like(out)
    for k in range(7):
        E.ed_execute(plan, w, ws if k % 2 == 0 else ws2, out if k % 2 == 0 else out2)
    torch.cuda.synchronize()
    assert torch.equal(ws.H(), ref_h) and torch.equal(out, ref_out)
    assert torch.equal(ws2.H()[: ref_h.shape[0]], ref_h) and torch.equal(out2, ref_out)
    ws2.release()
    ws3 = E.Workspace(plan)  # may reuse ws2's address: must bind afresh
    out3 = torch.zeros_like(out)
    for _ in range(3):
        E.ed_execute(plan, w, ws3, out3)
    torch.cuda.synchronize()
    assert torch.equal(out3, ref_out)
    err = compare(wl, plan, ws3, out3)
    assert all(v <= TOL[wl.dtype] for v in err.values()), err


def test_out_root_is_validated():
    from paper_2302_03851_b200 import edbatch as E
    wl = W.treelstm(4, (2, 6), 64, "bf16", cfg=73)
    plan, w, ws, out = run_gpu(wl)
    with pytest.raises(ValueError):
        E.ed_execute(plan, w, ws, out.float())
    with pytest.raises(ValueError):
        E.ed_execute(plan, w, ws, out[:2])


@pytest.mark.parametrize("h", [1024, 768, 320])
def test_treelstm_bf16_large_and_odd_hidden(h):
    """Hidden sizes past the bench's: h = 1024 (K = 2048, the bias no longer fits the shared-memory
    staging and is read from global), h = 768 and 320 (column tiles that do not divide h)."""
    _check(W.treelstm(12, (1, 24), h, "bf16", cfg=80 + h))


def test_lattice_h512_and_bilstm_h512():
    _check(W.lattice(16, (1, 30), 512, "bf16", cfg=84))
    _check(W.bilstm(10, (1, 20), 512, "bf16", cfg=85))


def test_minibatch_of_only_external_roots_and_one_op():
    """Degenerate minibatches: TreeFC instances that are single words (no op; the output is the input
    row) mixed with one one-op instance, and a minibatch with no op at all."""
    wl = W.treefc(1, (2, 2), 64, "bf16", cfg=86)
    words = [W.Graph(np.zeros(0, np.int32), np.zeros(1, np.int32), np.zeros(0, np.int32), np.zeros(0, np.int32), -1 - k)
             for k in (3, 9, 17)]
    wl.graphs = words + wl.graphs
    _check(wl)
    wl.graphs = words
    _check(wl)


@pytest.mark.parametrize("grid_max", ["64", "22"])
def test_split_k_pairs_with_several_tiles_per_cta(grid_max, monkeypatch):
    """Split-K pairs (A-28) when a batch has more tile pairs than CTA pairs: with the
    persistent grid capped (ED_GRID_MAX) every CTA exchanges partial sums for several tiles of one
    batch in turn (the xfree / xfull phases alternate within the batch).  TreeLSTM and TreeGRU
    forests at h = 512, where the small batches are split."""
    monkeypatch.setenv("ED_GRID_MAX", grid_max)
    for cell in ("treelstm", "treegru"):
        wl = W.treelstm(24, (2, 30), 512, "bf16", cfg=95, cell=cell)
        plan, _, _, _, _ = _check(wl)
        assert plan.info["split_steps"] > 0
        assert plan.query_info()["grid"] == int(grid_max)


def test_side_stream_uploads_into_two_workspaces_match_serial():
    """ed_io_t.upload_stream (the serving loop's overlap): a sequence of different minibatch plans
    executed in turn on two workspaces, each binding upload on a side stream ordered after the
    workspace's previous launch, gives the bitwise-same instance outputs as executing each plan
    alone on a fresh workspace with everything on one stream."""
    from paper_2302_03851_b200 import edbatch as E
    wls = [W.treelstm(30 + 4 * k, (2, 24), 256, "bf16", cfg=80 + k) for k in range(6)]
    ref = []
    for wl in wls:
        plan, w, ws, out = run_gpu(wl)
        ref.append(out.clone())
    ws_w = [E.DeviceWeights(wl.types, wl.params) for wl in wls]
    plans = [E.ed_plan(wl.graphs, wl.types, E.fsm_from_priority(wl.priority, len(wl.types))) for wl in wls]
    big = max(plans, key=lambda p: p.info["workspace_bytes"])
    wss = [E.Workspace(big), E.Workspace(big)]
    up = torch.cuda.Stream()
    outs = [torch.zeros_like(r) for r in ref]
    for rep in range(2):
        for k, (plan, o) in enumerate(zip(plans, outs)):
            E.ed_execute(plan, ws_w[k], wss[k % 2], o, upload_stream=up)
    torch.cuda.synchronize()
    for o, r in zip(outs, ref):
        assert torch.equal(o, r)


def test_split_disabled_and_enabled_both_match_the_oracle(monkeypatch):
    """The split-K pairs change only the fp32 summation order (A-28): with ED_SPLIT=0 (no clusters,
    one CTA per tile) and with the default both paths meet the parity tolerance, and they differ
    from each other by less than it."""
    wl = W.treelstm(16, (2, 30), 512, "bf16", cfg=96)
    monkeypatch.setenv("ED_SPLIT", "0")
    plan0, _, _, out0, _ = _check(wl)
    assert plan0.info["split_steps"] == 0
    monkeypatch.setenv("ED_SPLIT", "1")
    plan1, _, _, out1, _ = _check(wl)
    assert plan1.info["split_steps"] > 0
    d = (out0.float() - out1.float()).abs().max().item()
    assert d <= TOL[wl.dtype]


def test_split_k_plan_with_simt_tagger_steps():
    """One plan mixing TreeLSTM trees (whose small internal batches run split-K over CTA pairs, so
    the kernel is a cluster launch) with BiLSTM-tagger chains (whose tagger output runs as SIMT
    steps reusing the shared memory the split-K exchange also uses): both families meet the oracle."""
    import dataclasses
    tl = W.treelstm(12, (2, 24), 256, "bf16", cfg=97)
    bl = W.bilstm(10, (4, 20), 256, "bf16", cfg=98)
    nt, nw = len(tl.types), len(tl.params)
    types = list(tl.types) + [dataclasses.replace(t, weight_set=t.weight_set + nw) for t in bl.types]
    graphs = list(tl.graphs) + [W.Graph(g.type + nt, g.in_off, g.in_idx, g.ext, g.root) for g in bl.graphs]
    prio = list(tl.priority) + [p + nt for p in bl.priority]
    wl = W.Workload("mixed", types, graphs, prio, list(tl.params) + list(bl.params), "bf16", 256)
    plan, _, _, _, _ = _check(wl)
    assert plan.info["split_steps"] > 0
