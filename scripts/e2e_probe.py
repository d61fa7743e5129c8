"""Where the end-to-end serving loop spends its time (development aid): plan throughput of the
host pool, host cost of ed_execute per step, and the loop with plans prepared in advance."""
import sys, time, os, statistics
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import torch
import workloads as W
from paper_2302_03851_b200 import edbatch as E
wl = W.config(sys.argv[1] if len(sys.argv) > 1 else "cfg3")
learned = E.ed_fsm_learn(wl.graphs, wl.types, merged=True)
fsm = learned.table
plan = E.ed_plan(wl.graphs, wl.types, fsm)
weights = E.DeviceWeights(wl.types, wl.params)
ws = E.Workspace(plan)
out = torch.zeros(len(wl.graphs), wl.hidden, dtype=torch.bfloat16, device="cuda")
batch = E.GraphBatch(wl.graphs)
N = 30
t0 = time.perf_counter(); [E.ed_plan(batch, wl.types, fsm) for _ in range(5)]; t1 = time.perf_counter()
print(f"ed_plan serial: {(t1 - t0) / 5 * 1e3:.2f} ms per minibatch")
workers = max(1, min(14, (os.cpu_count() or 1) - 2))
pipe = E.PlanPipeline(wl.types, fsm, workers)
t0 = time.perf_counter(); futs = [pipe.submit(batch) for _ in range(N)]; plans = [f.result() for f in futs]; t1 = time.perf_counter()
print(f"ed_plan pool of {workers}: {(t1 - t0) / N * 1e6:.0f} us per minibatch")
host_out = [torch.empty(out.shape, dtype=out.dtype, pin_memory=True) for _ in range(2)]
for p in plans[:3]:
    ws.plan_info = p.info; E.ed_execute(p, weights, ws, out)
torch.cuda.synchronize()
ex = []
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
t0 = time.perf_counter()
for k, p in enumerate(plans):
    ws.plan_info = p.info
    s0 = time.perf_counter()
    E.ed_execute(p, weights, ws, out)
    ex.append(time.perf_counter() - s0)
    host_out[k % 2].copy_(out, non_blocking=True)
t1 = time.perf_counter()
b.record(); torch.cuda.synchronize()
print(f"prepared plans: host loop {(t1 - t0) / N * 1e6:.0f} us per step (ed_execute median {statistics.median(ex) * 1e6:.0f} us), "
      f"device {a.elapsed_time(b) / N * 1e3:.0f} us per step")
# same plan re-executed (no upload): the kernel + D2H only
a.record()
for k in range(N):
    E.ed_execute(plan, weights, ws, out)
    host_out[k % 2].copy_(out, non_blocking=True)
b.record(); torch.cuda.synchronize()
print(f"one plan re-executed: {a.elapsed_time(b) / N * 1e3:.0f} us per step")
pipe.close()
