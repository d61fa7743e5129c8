"""Per-CTA tile end times of the first device step (build with -DED_LEAF_TRACE; development aid)."""
import sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np, torch
import workloads as W
from harness import run_gpu
from paper_2302_03851_b200 import edbatch as E
wl = W.config(sys.argv[1] if len(sys.argv) > 1 else "cfg3")
plan, w, ws, out = run_gpu(wl)
nb = plan.info["num_steps"]
tr = torch.zeros(nb * 64 + 148 * 4, dtype=torch.int64, device="cuda")
for _ in range(3):
    tr.zero_()
    E.ed_execute(plan, w, ws, out, trace=tr)
torch.cuda.synchronize()
full = tr.cpu().numpy().astype(np.int64)
i = ws.plan_info
ts = ws._view(i["off_ts"], nb + 1, torch.int64).cpu().numpy().astype(np.int64)
t0 = ts[0]
pc = full[nb * 64:].reshape(148, 4)
print("step ends (us):", [round((x - t0) / 1e3, 1) for x in np.maximum.accumulate(ts[1:])][:4])
for k in range(4):
    v = pc[:, k][pc[:, k] > 0]
    if len(v): print(f"tile {k}: n={len(v)} end min/med/max us = {(v.min()-t0)/1e3:.1f} {(np.median(v)-t0)/1e3:.1f} {(v.max()-t0)/1e3:.1f}")
order = np.argsort(-pc.max(1))[:10]
print("slowest CTAs:", [(int(c), [round((x - t0) / 1e3, 1) if x else None for x in pc[c]]) for c in order])
