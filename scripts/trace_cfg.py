"""Per-phase trace of CTA 0 for each batch of a config (development aid)."""
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
tr = torch.zeros(nb * 64, dtype=torch.int64, device="cuda")
for _ in range(3):
    E.ed_execute(plan, w, ws, out, trace=tr)
torch.cuda.synchronize()
t = tr.view(nb, 64).cpu().numpy().astype(np.int64)
sched = plan.schedule()
print("phase stamps relative to step start (ns): [A-tab, A-issued, MMA-first-full, MMA-done, EPI-start, EPI-done, step-end]")
for s in range(nb):
    rel = [(int(t[s, k] - t[s, 0]) if t[s, k] else -1) for k in range(1, 8)]
    print(s, wl.types[sched[s][0]].name, len(sched[s][1]), rel)
for s in (1, 8, 13):
    base = t[s, 0]
    rel = lambda a, b: [int(t[s, k] - base) if t[s, k] else -1 for k in range(a, b)]
    print(f"step {s}: MMA full-wait done per kc:", rel(8, 24))
    print(f"step {s}: B issue per kc          :", rel(24, 40))
    print(f"step {s}: A release per kc        :", rel(40, 56))
print("step times:", ws.step_times_ns().tolist())
