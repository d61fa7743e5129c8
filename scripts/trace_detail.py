"""Detailed phase trace of item 0 of selected device steps (development aid): per-stage full
times of the MMA thread, per-stage issue times of loader thread 0, epilogue pass times.
Times in ns relative to the end of the previous step."""
import sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np, torch
import workloads as W
from harness import run_gpu
from paper_2302_03851_b200 import edbatch as E
name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
wl = W.config(name)
plan, w, ws, out = run_gpu(wl)
nb = plan.info["num_steps"]
tr = torch.zeros(nb * 64 + 148 * 4, dtype=torch.int64, device="cuda")
for _ in range(3):
    tr.zero_()
    E.ed_execute(plan, w, ws, out, trace=tr)
torch.cuda.synchronize()
full = tr.cpu().numpy().astype(np.int64)
t = full[:nb * 64].reshape(nb, 64)
i = ws.plan_info
ts = ws._view(i["off_ts"], nb + 1, torch.int64).cpu().numpy().astype(np.int64)
end = np.maximum.accumulate(ts)
sched = plan.schedule()
for s in range(nb):
    base = end[s]
    rel = lambda k: int(t[s, k] - base) if t[s, k] else None
    print(f"step {s} m={len(sched[min(s, len(sched) - 1)][1])} end={int(ts[s + 1] - base)}")
    print("  reached/rows-ready/A-issued/1st-full/MMA-issued/EPI-pre/EPI-acc/loop/fence/publish/EPI-done:",
          [rel(k) for k in (0, 1, 2, 3, 4, 7, 6, 8, 9, 10, 5)])
    print("  A stage free:", [rel(k) for k in range(48, 64) if t[s, k]])
    print("  B stage free:", [rel(k) for k in range(11, 27) if t[s, k]])
    print("  stage full:  ", [rel(k) for k in range(32, 48) if t[s, k]])
    print("  chunk4 A: loop-top/after-tma/pre-arrive/post-arrive:", [rel(k) for k in range(27, 31)])
    if t[s, 14]:
        print("  split exchange: partner-ld/xfree/sent/xfull:", [rel(k) for k in (14, 15, 16, 17)])
