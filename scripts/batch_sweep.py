"""Secondary report: instances/s of the device path versus minibatch size, for the
TreeLSTM h=512 workload of cfg3 (the paper reports its best over batch sizes 1-256).
Device time only (CUDA events around ed_execute, L2 flushed between runs), learned FSM.
    python scripts/batch_sweep.py [cell] > sweep.json"""
import json
import sys

sys.path.insert(0, ".")
import torch

import workloads as W
from paper_2302_03851_b200 import edbatch as E

cell = sys.argv[1] if len(sys.argv) > 1 else "treelstm"
flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device="cuda")
rows = []
for n in (1, 8, 32, 64, 128, 256, 512, 1024, 2048, 4096):
    wl = W.treelstm(n, (5, 40), 512, "bf16", 3, cell=cell)
    learned = E.ed_fsm_learn(wl.graphs, wl.types, merged=True)
    plan = E.ed_plan(wl.graphs, wl.types, learned.table)
    w = E.DeviceWeights(wl.types, wl.params)
    ws = E.Workspace(plan)
    out = torch.zeros(n, 512, dtype=torch.bfloat16, device="cuda")
    for _ in range(3):
        E.ed_execute(plan, w, ws, out)
    ts = []
    for _ in range(10):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        E.ed_execute(plan, w, ws, out)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = sorted(ts)[len(ts) // 2]
    rows.append({"instances": n, "nodes": wl.num_nodes, "batches": plan.info["num_batches"],
                 "us_per_pass": round(ms * 1e3, 1), "instances_per_s": round(n / (ms / 1e3))})
    print(json.dumps(rows[-1]), flush=True)
