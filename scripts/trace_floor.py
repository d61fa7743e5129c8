"""Phase trace of the latency-floor chain (bench.latency_floor_us): a caterpillar TreeLSTM h=512 with
24 dependent one-row internal steps.  Prints, per step, the item-0 CTA's phases relative to the
previous step's end (ns): reached, rows-ready, A-issued, MMA-1st-full, MMA-issued, EPI-got-acc,
EPI-done | step end."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import workloads as W
from paper_2302_03851_b200 import edbatch as E

wl = W.config("cfg3")
types, ins, ext = [0], [[]], [1]
prev = 0
for k in range(24):
    types.append(0); ins.append([]); ext.append(2 + k)
    leaf = len(types) - 1
    types.append(1); ins.append([prev, leaf]); ext.append(-1)
    prev = len(types) - 1
g = W.graph_from_lists(types, ins, ext, root=prev)
plan = E.ed_plan([g], wl.types[:2], E.fsm_from_priority([0, 1], 2))
w = E.DeviceWeights(wl.types[:2], wl.params[:2])
ws = E.Workspace(plan)
out = torch.zeros(1, 512, dtype=torch.bfloat16, device="cuda")
nb = plan.info["num_steps"]
tr = torch.zeros(nb * 64 + 148 * 4, dtype=torch.int64, device="cuda")
for _ in range(4):
    tr.zero_()
    E.ed_execute(plan, w, ws, out, trace=tr)
torch.cuda.synchronize()
t = tr.cpu().numpy().astype(np.int64)[:nb * 64].reshape(nb, 64)
i = ws.plan_info
ts = ws._view(i["off_ts"], nb + 1, torch.int64).cpu().numpy().astype(np.int64)
end = np.maximum.accumulate(ts)
for s in range(nb):
    base = end[s]
    rel = lambda k: int(t[s, k] - base) if t[s, k] else None
    print(s, [rel(k) for k in (0, 1, 2, 3, 4, 6, 10, 11, 12, 13, 7, 8, 9, 5)], "|", int(ts[s + 1] - base))
    if len(sys.argv) > 1:
        print("   mma", [rel(k) for k in range(24, 32)])
