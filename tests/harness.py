"""Test helpers: run a workload through the C ABI and compare with the fp64 oracle.

Test infrastructure (may import oracle/).  Tolerance metric (reading A-19): per output
tensor max_i |y_i - r_i| / max(max_i |r_i|, 1e-6).
"""
from __future__ import annotations

import numpy as np
import torch

from oracle.evaluate import evaluate_recursive, root_outputs
from oracle.graph import Merged

TOL = {"fp32": 1e-4, "bf16": 2e-2}


def rel_err(y: np.ndarray, r: np.ndarray) -> float:
    y = np.asarray(y, np.float64)
    r = np.asarray(r, np.float64)
    return float(np.max(np.abs(y - r)) / max(float(np.max(np.abs(r))), 1e-6)) if r.size else 0.0


def run_gpu(wl, layout=0, priority=None, stream=None, staging=0, fsm=None):
    from paper_2302_03851_b200 import edbatch as E
    pr = wl.priority if priority is None else priority
    table = fsm if fsm is not None else E.fsm_from_priority(pr, len(wl.types))
    plan = E.ed_plan(wl.graphs, wl.types, table, layout=layout, staging=staging)
    w = E.DeviceWeights(wl.types, wl.params)
    ws = E.Workspace(plan)
    dt = torch.bfloat16 if wl.dtype == "bf16" else torch.float32
    out = torch.zeros(len(wl.graphs), wl.hidden, dtype=dt, device="cuda")
    E.ed_execute(plan, w, ws, out)
    torch.cuda.synchronize()
    return plan, w, ws, out


def compare(wl, plan, ws, out, instances=None):
    """Element-by-element comparison of every node record (h, c, logits) and the root outputs
    for the given instances (default: all).  Returns dict of errors per tensor kind."""
    idx = list(range(len(wl.graphs))) if instances is None else list(instances)
    recs = evaluate_recursive(wl, idx)
    m = Merged(wl.graphs, len(wl.types))
    row = plan.layout()
    H = ws.H().float().cpu().numpy()
    C = ws.C().cpu().numpy()
    Y = ws.Y().cpu().numpy() if plan.info["y_cols"] else None
    X = ws.X().cpu().numpy() if ws.X() is not None else None
    Mx = ws.M()   # MV-RNN node matrices, stored transposed (compared when small enough to copy)
    Mx = Mx.float().cpu().numpy() if Mx is not None and Mx.numel() <= (1 << 27) else None
    ys, rs = {"h": [], "c": [], "y": [], "l": [], "M": []}, {"h": [], "c": [], "y": [], "l": [], "M": []}
    for k, gi in enumerate(idx):
        base = m.base[gi]
        for v, rec in recs[k].items():
            r = row[base + v]
            if rec.get("h") is not None:
                ys["h"].append(H[r]); rs["h"].append(rec["h"])
            if rec.get("c") is not None:
                ys["c"].append(C[r]); rs["c"].append(rec["c"])
            if rec.get("M") is not None and Mx is not None:
                ys["M"].append(Mx[r].T.ravel()); rs["M"].append(np.asarray(rec["M"]).ravel())
            if rec.get("l") is not None:
                ys["l"].append(X[r]); rs["l"].append(rec["l"])
            if rec.get("y") is not None:
                C_ = len(rec["y"])
                ys["y"].append(Y[r][:C_]); rs["y"].append(rec["y"])
    err = {k: rel_err(np.concatenate(ys[k]), np.concatenate(rs[k])) for k in ys if ys[k]}
    root_ref = root_outputs(wl, recs, idx)
    err["root"] = rel_err(out.float().cpu().numpy()[idx], root_ref)
    return err
