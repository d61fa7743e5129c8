"""Quick GPU check: parity of several workloads and a timing of cfg3 (development aid)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import workloads as W
from harness import run_gpu, compare, TOL

cases = [
    ("cfg1 treelstm h32 fp32", lambda: W.config("cfg1"), None),
    ("treelstm h64 bf16", lambda: W.treelstm(12, (2, 20), 64, "bf16", 7), None),
    ("treelstm h128 bf16", lambda: W.treelstm(40, (2, 30), 128, "bf16", 8), None),
    ("treelstm h512 bf16 (16 trees)", lambda: W.treelstm(16, (5, 40), 512, "bf16", 3), None),
]
for name, f, inst in cases:
    wl = f()
    t0 = time.time()
    try:
        plan, w, ws, out = run_gpu(wl)
        err = compare(wl, plan, ws, out, inst)
        ok = all(v <= TOL[wl.dtype] for v in err.values())
        print(f"{name}: {'OK' if ok else 'FAIL'} {err} ({time.time()-t0:.1f}s)", flush=True)
    except Exception as e:
        print(f"{name}: EXC {e}", flush=True)
        import traceback; traceback.print_exc()

# timing cfg3
from paper_2302_03851_b200 import edbatch as E
wl = W.config("cfg3")
plan, w, ws, out = run_gpu(wl)
err = compare(wl, plan, ws, out, list(range(0, 256, 16)))
print("cfg3 parity (16 sampled trees):", err, flush=True)
for _ in range(3):
    E.ed_execute(plan, w, ws, out)
torch.cuda.synchronize()
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record()
N = 20
for _ in range(N):
    E.ed_execute(plan, w, ws, out)
ev1.record(); torch.cuda.synchronize()
ms = ev0.elapsed_time(ev1) / N
print(f"cfg3: {ms*1e3:.1f} us/pass, {256/ms*1e3:.0f} inst/s; steps(ns):", ws.step_times_ns().tolist(), flush=True)
