"""Run a config a few times through the C ABI (for ncu / compute-sanitizer captures)."""
import sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import torch
import workloads as W
from harness import run_gpu
from paper_2302_03851_b200 import edbatch as E
name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
layout = int(sys.argv[3]) if len(sys.argv) > 3 else 0
wl = W.config(name)
plan, w, ws, out = run_gpu(wl, layout=layout)
for _ in range(reps):
    E.ed_execute(plan, w, ws, out)
torch.cuda.synchronize()
print("steps(ns):", ws.step_times_ns().tolist())
