"""GPU parity at every size bench.py reports, in bench.py's launch configuration.

bench.py plans each config with the FSM table Q-learned over the merged minibatch (PAPER §2.3,
ed_fsm_learn merged episodes), the schedule-order layout and producer staging (S-1); the
column-tile geometry of every batch depends on h and m, so each benched (cell, h, minibatch) gets
its own launch-shape check here.  The fp64 oracle evaluates a sample of instances (the 8 tallest
plus random ones, SURVEY O-5 subset trick) and those rows of the full GPU run are compared element
by element (tolerance metric A-19, 2e-2 for bf16).

Also the sharded path on one GPU: the LPT shards of a minibatch planned and
executed one after another give roots bitwise equal to the unsharded run.
"""
import numpy as np
import pytest
import torch

import workloads as W
from harness import TOL, compare

pytestmark = pytest.mark.gpu


def bench_plan(wl):
    """The plan bench.py times: learned (merged episodes) FSM, schedule layout, staging auto."""
    from paper_2302_03851_b200 import edbatch as E
    learned = E.ed_fsm_learn(wl.graphs, wl.types, merged=True)
    return E.ed_plan(wl.graphs, wl.types, learned.table, layout=E.ED_LAYOUT_SCHEDULE_ORDER,
                     staging=E.ED_STAGING_AUTO)


def run_plan(wl, plan):
    from paper_2302_03851_b200 import edbatch as E
    w = E.DeviceWeights(wl.types, wl.params)
    ws = E.Workspace(plan)
    dt = torch.bfloat16 if wl.dtype == "bf16" else torch.float32
    out = torch.zeros(len(wl.graphs), wl.hidden, dtype=dt, device="cuda")
    E.ed_execute(plan, w, ws, out)
    torch.cuda.synchronize()
    return w, ws, out


def sample(wl, n_random, seed=11):
    sizes = [g.num_nodes for g in wl.graphs]
    tallest = [int(i) for i in np.argsort(sizes, kind="stable")[-8:]]
    rng = np.random.default_rng(seed)
    rest = [int(i) for i in rng.choice(len(wl.graphs), n_random, replace=False)]
    return sorted(set(tallest + rest))


@pytest.mark.parametrize("name,n_random", [
    ("cfg3", 24), ("cfg3_gru", 24), ("cfg3_2type", 24), ("cfg4_treefc", 48), ("cfg2", 16),
    ("cfg5", 32), ("cfg5_gru", 32), ("cfg5_h512", 24),
])
def test_bench_config_full_size_sampled(name, n_random):
    wl = W.config(name)
    plan = bench_plan(wl)
    w, ws, out = run_plan(wl, plan)
    err = compare(wl, plan, ws, out, sample(wl, n_random))
    assert all(v <= TOL[wl.dtype] for v in err.values()), err


@pytest.mark.parametrize("split", ["0", "1"])
@pytest.mark.parametrize("name,world", [("cfg3", 4), ("cfg5", 8)])
def test_lpt_shards_run_sequentially_equal_unsharded_bitwise(name, world, split, monkeypatch):
    """Instances are independent: each node's value depends only on its own inputs, so the
    per-rank plans of the LPT partition reproduce the unsharded roots bit for bit.
    With split-K over CTA pairs (ED_SPLIT=1, the default) whether a batch is split depends on its
    size, and a split tile adds its two K halves' fp32 partial sums (a different rounding order
    than one accumulation over K, reading A-28): the shards then agree with the
    unsharded run to the parity tolerance instead of bitwise."""
    from paper_2302_03851_b200.sharding import lpt_partition
    monkeypatch.setenv("ED_SPLIT", split)
    wl = W.config(name)
    _, _, full = run_plan(wl, bench_plan(wl))
    got = torch.zeros_like(full)
    parts = lpt_partition([g.num_nodes for g in wl.graphs], world)
    assert sorted(i for p in parts for i in p) == list(range(len(wl.graphs)))
    for idx in parts:
        sub = W.Workload(name=wl.name, types=wl.types, graphs=[wl.graphs[i] for i in idx], priority=wl.priority,
                         params=wl.params, dtype=wl.dtype, hidden=wl.hidden, config=wl.config)
        _, _, out = run_plan(sub, bench_plan(sub))
        got[idx] = out
    if split == "0":
        assert torch.equal(got, full)
    else:
        d = (got.float() - full.float()).abs()
        assert float(d.max()) <= TOL[wl.dtype] * max(1.0, float(full.float().abs().max())), float(d.max())


def test_split_k_steps_present_and_pairs_resident():
    """cfg3's small batches (<= half a wave of 16-unit tiles) run split-K over CTA pairs, and the
    cluster launch keeps one CTA per SM on all 148 SMs (every pair co-resident: dataflow waits)."""
    from paper_2302_03851_b200 import edbatch as E
    wl = W.config("cfg3")
    plan = bench_plan(wl)
    assert plan.info["split_steps"] >= 5
    run_plan(wl, plan)
    g = plan.query_info()["grid"]
    assert g % 2 == 0 and g >= 140, g
