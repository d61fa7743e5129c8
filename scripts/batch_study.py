"""Batch-count study (PAPER Fig. 8): batches the policies execute on the merged BASELINE
minibatches, through the product planner only (ed_plan policies + ed_fsm_learn encoders), with the
App. B.3 lower bound, and -- with a GPU -- the device time of one pass of each schedule.

    python scripts/batch_study.py [--gpu] [--out profiles/batch_study_r02]

Policies: TF-Fold depth-based, DyNet agenda-based, the sufficient-condition heuristic (argmax of
Eq. 1's second term), and the FSM learned by Q-learning over the merged minibatch with each state
encoding E_base / E_max / E_sort.
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as W  # noqa: E402
from paper_2302_03851_b200 import edbatch as E  # noqa: E402

CONFIGS = ["cfg2", "cfg3", "cfg3_2type", "cfg4_treefc", "cfg5", "cfg5_gru"]


def device_us(plan, wl, weights, reps=7):
    import torch
    ws = E.Workspace(plan)
    dt = torch.bfloat16 if wl.dtype == "bf16" else torch.float32
    out = torch.zeros(len(wl.graphs), wl.hidden, dtype=dt, device="cuda")
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device="cuda")
    for _ in range(3):
        E.ed_execute(plan, weights, ws, out)
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        E.ed_execute(plan, weights, ws, out)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    ws.release()
    return statistics.median(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpu", action="store_true")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "batch_study_r02"))
    args = ap.parse_args()
    rows = []
    for name in CONFIGS:
        wl = W.config(name)
        weights = E.DeviceWeights(wl.types, wl.params) if args.gpu else None
        plans = {}
        for pol, code in (("depth", E.ED_POLICY_DEPTH), ("agenda", E.ED_POLICY_AGENDA), ("sc", E.ED_POLICY_SC)):
            plans[pol] = E.ed_plan(wl.graphs, wl.types, [], policy=code)
        for enc, code in (("fsm_base", E.ED_ENC_BASE), ("fsm_max", E.ED_ENC_MAX), ("fsm_sort", E.ED_ENC_SORT)):
            learned = E.ed_fsm_learn(wl.graphs, wl.types, encoder=code, merged=True)
            plans[enc] = E.ed_plan(wl.graphs, wl.types, learned.table, encoder=code)
        row = {"config": name, "instances": len(wl.graphs), "nodes": wl.num_nodes,
               "lower_bound": plans["depth"].info["lower_bound"],
               "batches": {k: p.info["num_batches"] for k, p in plans.items()}}
        if args.gpu:
            row["device_us"] = {k: round(device_us(p, wl, weights), 1) for k, p in plans.items()}
        rows.append(row)
        print(json.dumps(row), flush=True)
    json.dump(rows, open(args.out + ".json", "w"), indent=1)
    keys = ["depth", "agenda", "sc", "fsm_base", "fsm_max", "fsm_sort"]
    with open(args.out + ".md", "w") as f:
        f.write("# Batch-count study (PAPER Fig. 8, P:434-436) on the merged BASELINE minibatches\n\n")
        f.write("Batches executed per pass (device us per pass in parentheses, L2 flushed, median of 7)."
                " FSM = Q-learned over the merged minibatch with the given state encoding (P:125).\n\n")
        f.write("| config | nodes | lower bound | " + " | ".join(keys) + " |\n|" + "---|" * (3 + len(keys)) + "\n")
        for r in rows:
            cells = []
            for k in keys:
                c = str(r["batches"][k])
                if "device_us" in r:
                    c += f" ({r['device_us'][k]:.0f} us)"
                cells.append(c)
            f.write(f"| {r['config']} | {r['nodes']} | {r['lower_bound']} | " + " | ".join(cells) + " |\n")


if __name__ == "__main__":
    main()
