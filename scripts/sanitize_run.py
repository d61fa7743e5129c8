"""One small execute per path for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
a bf16 TreeLSTM forest (tensor-core path, staged + gathered operands, several tiles, split-K
pairs), a bf16 lattice minibatch (variadic word inputs, link gates), a TreeLSTM forest at h = 512
(split-K pairs over clusters of 2, DSMEM exchange), a BiLSTM tagger (LSTM cells + SIMT tagger
output) and the fp32 cfg1 TreeLSTM (SIMT path).
Exits non-zero if an output misses the oracle tolerance."""
import sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import torch
import workloads as W
from harness import TOL, compare, run_gpu

ok = True
for wl in (W.treelstm(20, (1, 24), 128, "bf16", cfg=91), W.lattice(12, (2, 20), 64, "bf16", cfg=92),
           W.treelstm(6, (2, 20), 512, "bf16", cfg=94),          # split-K pairs at h = 512 (clusters of 2)
           W.bilstm(8, (4, 20), 64, "bf16", cfg=93),             # LSTM + tagger SIMT steps
           W.config("cfg1")):
    plan, w, ws, out = run_gpu(wl)
    err = compare(wl, plan, ws, out)
    good = all(v <= TOL[wl.dtype] for v in err.values())
    ok &= good
    print(wl.name, plan.info["num_batches"], "batches", err, "OK" if good else "FAIL", flush=True)
torch.cuda.synchronize()
sys.exit(0 if ok else 1)
