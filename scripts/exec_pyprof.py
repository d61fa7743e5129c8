import sys, time
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import torch, ctypes
import workloads as W
from paper_2302_03851_b200 import edbatch as E
wl = W.config("cfg3")
learned = E.ed_fsm_learn(wl.graphs, wl.types, merged=True)
plans = [E.ed_plan(wl.graphs, wl.types, learned.table) for _ in range(12)]
weights = E.DeviceWeights(wl.types, wl.params)
ws = E.Workspace(plans[0])
out = torch.zeros(len(wl.graphs), wl.hidden, dtype=torch.bfloat16, device="cuda")
for p in plans[:2]: E.ed_execute(p, weights, ws, out)
torch.cuda.synchronize()
def t(f, n=200):
    t0 = time.perf_counter()
    for _ in range(n): f()
    return (time.perf_counter() - t0) / n * 1e6
print("current_stream", t(lambda: torch.cuda.current_stream()))
print("_stream_handle", t(lambda: E._stream_handle(None)))
print("checks", t(lambda: (out.is_cuda and out.is_contiguous() and out.dtype == torch.bfloat16 and out.numel())))
print("data_ptr", t(lambda: out.data_ptr()))
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
for p in plans[2:]:
    E.ed_execute(p, weights, ws, out)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(8)
ts=[]
for p in plans[2:]:
    s0=time.perf_counter(); E.ed_execute(p, weights, ws, out); ts.append(time.perf_counter()-s0)
print("ed_execute per call us", [round(x*1e6) for x in ts])
