#!/usr/bin/env python
"""bench.py — ED-Batch hot path (arXiv 2302.03851) on B200: instances/s of one full batched
forward pass (every batch of the FSM schedule) over a minibatch of synthetic instance graphs.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg3] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (one process per GPU)

A "step" is one ed_execute (one persistent kernel) over the minibatch (BASELINE cfg3: 256
TreeLSTM trees, h = 512, bf16), inputs resident in HBM; L2 (126 MB) is flushed between timed
steps by a 256 MB write.  Multi-GPU: instances are sharded, every rank runs its own minibatch of
the same size (weak scaling) with no data-path collective; time = max over ranks.
Prints ONE JSON line (rank 0).  DESIGN.md §7 documents every field.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

METRIC = "instances/sec TreeLSTM h=512 (BASELINE cfg3: 256 random trees, bf16) per step, whole job"
METRICS = {"cfg3": METRIC,
           "cfg3_gru": "instances/sec TreeGRU h=512 (256 random trees, bf16) per step, whole job",
           "cfg3_2type": "instances/sec TreeLSTM-2Type h=512 (256 random trees, bf16) per step, whole job",
           "cfg1": "instances/sec TreeLSTM h=32 (cfg1: 8 random trees, fp32) per step, whole job",
           "cfg2": "instances/sec BiLSTM-tagger h=256 (cfg2: 64 sequences, bf16) per step, whole job",
           "cfg5": "instances/sec LatticeLSTM h=256 (cfg5: 512 lattices, bf16) per step, whole job",
           "cfg5_h512": "instances/sec LatticeLSTM h=512 (512 lattices, bf16; BASELINE metric, A-24) per step, whole job",
           "cfg5_gru": "instances/sec LatticeGRU h=256 (512 lattices, bf16) per step, whole job",
           "cfg4_treefc": "instances/sec TreeFC h=512 (cfg4: 1024 trees, bf16) per step, whole job",
           "cfg4_mvrnn": "instances/sec MV-RNN h=512 (cfg4: 1024 trees, bf16) per step, whole job"}
CONFIGS = {
    "cfg3": "cfg3 TreeLSTM h=512, 256 parse-like random binary trees (leaves U[5,40]), bf16",
    "cfg3_gru": "cfg3 TreeGRU h=512, 256 parse-like random binary trees (leaves U[5,40]), bf16",
    "cfg3_2type": "cfg3 TreeLSTM-2Type h=512 (two internal types 50/50, P:291), 256 random trees (leaves U[5,40]), bf16",
    "cfg1": "cfg1 TreeLSTM h=32, 8 random trees (leaves U[2,16]), fp32",
    "cfg2": "cfg2 BiLSTM tagger h=256, 64 sequences of length U[10,50], bf16",
    "cfg5": "cfg5 LatticeLSTM h=256, 512 character lattices (chars U[10,50], word p=0.3), bf16",
    "cfg5_h512": "cfg5 LatticeLSTM h=512 (the metric's hidden size, A-24), 512 character lattices (chars U[10,50], word p=0.3), bf16",
    "cfg5_gru": "cfg5 LatticeGRU h=256 (P:294, A-27), 512 character lattices (chars U[10,50], word p=0.3), bf16",
    "cfg4_treefc": "cfg4 TreeFC h=512, 1024 random trees (leaves U[5,40]), bf16",
    "cfg4_mvrnn": "cfg4 MV-RNN h=512, 1024 random trees (leaves U[5,40], 1024 word vectors + matrices), bf16",
}


def make_workload(name: str, rank: int, world: int = 1, scaling: str = "weak"):
    """weak: every rank runs its own minibatch of the config's size (rank 0 = the exact config);
    strong: the config's minibatch is LPT-sharded across ranks by node count."""
    if scaling == "strong":
        from paper_2302_03851_b200.sharding import shard_graphs
        wl = W.config(name)
        n_total = len(wl.graphs)
        wl.shard_idx, wl.graphs = shard_graphs(wl.graphs, rank, world)
        wl.n_total = n_total
        return wl
    wl = _weak_workload(name, rank)
    wl.shard_idx = [rank * len(wl.graphs) + i for i in range(len(wl.graphs))]   # global instance ids
    wl.n_total = world * len(wl.graphs)
    return wl


def _weak_workload(name: str, rank: int):
    if rank == 0:
        return W.config(name)
    if name == "cfg3_2type":
        return W.treelstm_2type(256, (5, 40), 512, "bf16", 3 + 100 * rank)
    if name in ("cfg3", "cfg3_gru"):
        return W.treelstm(256, (5, 40), 512, "bf16", 3 + 100 * rank, cell="treegru" if name == "cfg3_gru" else "treelstm")
    if name == "cfg1":
        return W.treelstm(8, (2, 16), 32, "fp32", 1 + 100 * rank)
    if name == "cfg2":
        return W.bilstm(64, (10, 50), 256, "bf16", 2 + 100 * rank)
    if name == "cfg5":
        return W.lattice(512, (10, 50), 256, "bf16", 5 + 100 * rank)
    if name == "cfg5_h512":
        return W.lattice(512, (10, 50), 512, "bf16", 5 + 100 * rank)
    if name == "cfg5_gru":
        return W.lattice(512, (10, 50), 256, "bf16", 5 + 100 * rank, cell="latticegru")
    if name == "cfg4_treefc":
        return W.treefc(1024, (5, 40), 512, "bf16", 4 + 100 * rank)
    if name == "cfg4_mvrnn":
        return W.treefc(1024, (5, 40), 512, "bf16", 4 + 100 * rank, cell="mvrnn")
    raise KeyError(name)


def host_cpu():
    """CPU model and logical core count of this host (lscpu), for the CPU baseline."""
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        model = next((l.split(":", 1)[1].strip() for l in out.splitlines() if l.startswith("Model name")), "?")
    except Exception:
        model = "?"
    return {"model": model, "logical_cpus": os.cpu_count()}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["bf16_tflops"]), float(d.get("bf16_tflops_sustained", d["bf16_tflops"])), float(d["hbm_gbs"]), "measured"
    return 1590.0, 1400.0, 6650.0, "fallback"


# --- algorithmic work per batch -----------------------------------
def step_work(kind: str, m: int, h: int, C: int, elt: int):
    """(flops, hbm bytes) of one batch of m ops, weights excluded."""
    if kind == "treelstm_leaf":
        return 2 * m * h * 3 * h, m * (elt * h + 4 + elt * h + 4 * h)
    if kind == "treelstm_internal":
        return 2 * m * 2 * h * 5 * h, m * (2 * elt * h + 2 * 4 * h + elt * h + 4 * h)
    if kind == "linear_out":
        return 2 * m * h * C, m * (elt * h + 4 * C)
    if kind == "treegru_leaf":
        return 2 * m * h * 2 * h, m * (elt * h + 4 + elt * h)
    if kind == "treegru_internal":
        return 2 * m * (2 * h * 3 * h + 2 * h * h), m * (2 * elt * h + elt * h)
    if kind == "treefc_internal":
        return 2 * m * 2 * h * h, m * (2 * elt * h + elt * h)
    if kind == "mvrnn_internal":
        # p = tanh(W [B a; A b] + b): 2 matvecs (2h^2 each) + K=2h GEMM; P = W_M [A; B]: 4h^3.
        # bytes: the two child matrices read once, P written, vectors
        return m * (2 * 2 * h * h + 2 * 2 * h * h + 4 * h * h * h), m * (3 * elt * h * h + 3 * elt * h + 2 * elt * h)
    if kind == "lstm":
        return 2 * m * 2 * h * 4 * h, m * (elt * h + 4 + elt * h + 4 * h + elt * h + 4 * h)
    if kind == "tagger":
        return 2 * m * 2 * h * h + 2 * m * h * C, m * (2 * elt * h + 4 * C)
    if kind == "lattice_char":
        return 2 * m * 2 * h * 4 * h, m * (elt * h + 4 + elt * h + 4 * h + elt * h + 4 * h)
    if kind == "lattice_word":
        return 2 * m * 2 * h * 3 * h + 2 * m * 2 * h * h, m * (elt * h + 4 + elt * h + 4 * h + elt * h + 4 * h + 4 * h)
    if kind in ("latticegru_char", "latticegru_word"):  # GRU over [x; h]: [r; z; n_x; n_h] (A-27)
        return 2 * m * 2 * h * 4 * h, m * (elt * h + 4 + elt * h + elt * h)
    raise KeyError(kind)


def weight_bytes(kind: str, h: int, C: int, elt: int) -> int:
    g = {"treelstm_leaf": (3, 1), "treelstm_internal": (5, 2), "treegru_leaf": (2, 1), "treegru_internal": (5, 2),
         "treefc_internal": (1, 2), "lstm": (4, 2), "tagger": (1, 2), "lattice_char": (4, 2), "lattice_word": (4, 2),
         "latticegru_char": (4, 2), "latticegru_word": (4, 2)}
    if kind == "linear_out":
        return 4 * C * h
    if kind == "tagger":
        return elt * 2 * h * h + 4 * h + 4 * C * h + 4 * C
    if kind == "mvrnn_internal":
        return 2 * elt * 2 * h * h + 4 * h   # W and W_M (word vectors/matrices: per-node bytes)
    G, S = g[kind]
    return elt * G * h * S * h + 4 * G * h


def plan_roofline(wl, plan, P_tflops, BW_gbs):
    """Per-batch roofline t_roof = max(F / P, B / BW); weights charged once per pass (first use)."""
    elt = 2 if wl.dtype == "bf16" else 4
    seen = set()
    F_tot = B_tot = 0
    troof = []
    for t, mem in plan.schedule():
        ot = wl.types[t]
        F, B = step_work(ot.kind, len(mem), wl.hidden, ot.out_dim, elt)
        if ot.weight_set not in seen:
            seen.add(ot.weight_set)
            B += weight_bytes(ot.kind, wl.hidden, ot.out_dim, elt)
        F_tot += F
        B_tot += B
        troof.append(max(F / (P_tflops * 1e12), B / (BW_gbs * 1e9)))
    return F_tot, B_tot, troof


# --- clocks ---------------------------------------------------------------------------------
class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self):
        self.proc = None

    def start(self):
        """Starts nvidia-smi and returns once it has printed its first sample, so the sampler is
        live for the whole timed region (a short region otherwise ends before nvidia-smi starts)."""
        self.first = ""
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        import select
        r, _, _ = select.select([self.proc.stdout], [], [], 5.0)
        if r:
            self.first = self.proc.stdout.readline()

    def stop(self, ngpu: int):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out, _ = self.proc.communicate()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in (self.first + (out or "")).strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9 or not f[0].isdigit() or int(f[0]) >= ngpu:
                continue
            try:
                sm.append(float(f[1])); mx.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons), "samples": len(sm)}


# --- CPU oracle baseline (bounded sample) -------------------------------------------------------
def latency_floor_us(E, wl, depth: int = 24):
    """SURVEY §8(d) latency floor: the per-step cost of the same persistent kernel on a chain of
    dependent one-row batches (a caterpillar tree of the workload's cell types: each internal node
    reads the previous one and a fresh leaf), i.e. readiness propagation + operand load + K chain +
    epilogue with no parallel work.  Median in-kernel step time of the internal steps.  Only for the
    tree workloads (L, I[, I2], O types)."""
    import numpy as np
    import torch
    names = [t.name for t in wl.types]
    if names[:2] != ["L", "I"] and names[:2] != ["L", "I1"]:
        return None
    types, ins, ext = [], [], []
    types.append(0); ins.append([]); ext.append(1)
    prev = 0
    for k in range(depth):
        types.append(0); ins.append([]); ext.append(2 + k)
        leaf = len(types) - 1
        types.append(1); ins.append([prev, leaf]); ext.append(-1)
        prev = len(types) - 1
    g = W.graph_from_lists(types, ins, ext, root=prev)
    plan = E.ed_plan([g], wl.types[:2], E.fsm_from_priority([0, 1], 2))
    weights = E.DeviceWeights(wl.types[:2], wl.params[:2])
    ws = E.Workspace(plan)
    out = torch.zeros(1, wl.hidden, dtype=torch.bfloat16 if wl.dtype == "bf16" else torch.float32, device="cuda")
    for _ in range(4):
        E.ed_execute(plan, weights, ws, out)
    torch.cuda.synchronize()
    st = ws.step_times_ns()
    return float(np.median(st[1:])) / 1e3 if len(st) > 2 else None


def cpu_oracle_rate(wl, seconds: float, max_instances: int = 256):
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle.evaluate import evaluate_recursive
    try:
        from threadpoolctl import threadpool_limits
        limiter = threadpool_limits(1)
    except Exception:  # pragma: no cover
        limiter = None
    n = 0
    t0 = time.perf_counter()
    while n < max_instances and time.perf_counter() - t0 < seconds:
        evaluate_recursive(wl, [n % len(wl.graphs)])
        n += 1
    dt = time.perf_counter() - t0
    if limiter is not None:
        limiter.unregister() if hasattr(limiter, "unregister") else None
    return n / dt, n, dt


_WORKER_WL = None


def _oracle_worker_init(name):
    global _WORKER_WL
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:  # pragma: no cover
        pass
    _WORKER_WL = W.config(name)


def _oracle_worker_eval(i):
    from oracle.evaluate import evaluate_recursive
    if i >= 0:
        evaluate_recursive(_WORKER_WL, [i % len(_WORKER_WL.graphs)])
    return i


def cpu_oracle_rate_all_cores(name, rate1: float, seconds: float):
    """The same fp64 oracle on every host core (1-thread and all-core rates): a
    process pool over instances (spawned workers, 1 BLAS thread each), a bounded sample sized from
    the 1-core rate.  Returns (instances/s, instances, seconds, cores)."""
    import concurrent.futures as cf
    import multiprocessing as mp
    cores = os.cpu_count() or 1
    n = max(cores, min(4096, int(rate1 * cores * seconds)))
    with cf.ProcessPoolExecutor(cores, mp_context=mp.get_context("spawn"), initializer=_oracle_worker_init,
                                initargs=(name,)) as ex:
        list(ex.map(_oracle_worker_eval, [-1] * cores))   # workers up and holding the workload
        t0 = time.perf_counter()
        list(ex.map(_oracle_worker_eval, range(n), chunksize=max(1, n // (4 * cores))))
        dt = time.perf_counter() - t0
    return n / dt, n, dt, cores


def run_reference(args, rank, world):
    """--impl reference: the fp64 oracle (plain per-node topological evaluation) on host cores,
    each step a bounded sample of the same workload; rank 0 only."""
    if rank != 0:
        return
    wl = make_workload(args.config, 0)
    sample = args.ref_sample
    from oracle.evaluate import evaluate_recursive
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:
        pass
    times = []
    for s in range(args.warmup + args.steps):
        idx = [(s * sample + k) % len(wl.graphs) for k in range(sample)]
        t0 = time.perf_counter()
        evaluate_recursive(wl, idx)
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            times.append(dt)
    ms = 1e3 * sum(times) / len(times)
    v = sample / (ms / 1e3)
    line = {"impl": "reference", "metric": METRICS[args.config], "value": v, "unit": "instances/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": CONFIGS[args.config], "sample_instances_per_step": sample},
            "cpu_baseline": {"value": v, "unit": "instances/s", "cores": 1, "kind": "oracle",
                             "sample": f"{sample} instances per step of the {args.config} minibatch, fp64 per-node "
                                       "recursive oracle (oracle/evaluate.py), 1 BLAS thread"},
            "e2e": {"value": v, "unit": "instances/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="cfg3", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--layout", default="schedule", choices=["schedule", "pq"])
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--staging", default="auto", choices=["auto", "off"])
    ap.add_argument("--step-order", default="level", choices=["level", "schedule"])
    ap.add_argument("--fsm", default="learned", choices=["learned", "learned_instance", "priority"])
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--ref-sample", type=int, default=8)
    ap.add_argument("--e2e-steps", type=int, default=300,
                    help="minibatches of the end-to-end serving loop (planning pipeline fill amortised over them)")
    ap.add_argument("--plan-threads", type=int, default=14, help="host threads planning minibatches ahead (e2e)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    # ED_BENCH_ONE_GPU=1 (test hook): every rank on cuda:0 over gloo, to exercise the N > 1 code path
    # (sharding, RootGather, max-over-ranks timing) on a one-GPU box; never used for reported numbers
    one_gpu = os.environ.get("ED_BENCH_ONE_GPU") == "1"
    if one_gpu:
        local = 0
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2302_03851_b200 import edbatch as E
    from paper_2302_03851_b200.sharding import RootGather

    wl = make_workload(args.config, rank, world, args.scaling)
    layout = E.ED_LAYOUT_PQ if args.layout == "pq" else E.ED_LAYOUT_SCHEDULE_ORDER
    fsm_info = {"fsm": args.fsm}
    if args.fsm.startswith("learned"):  # PAPER §2.3: Q-learned per topology, offline, not timed
        # episodes over the merged minibatch (the graph ed_plan schedules) unless learned_instance
        learned = E.ed_fsm_learn(wl.graphs, wl.types, merged=args.fsm == "learned")
        fsm = learned.table
        fsm_info.update(fsm_episodes=learned.info["episodes"], fsm_learn_ms=round(learned.info["learn_us"] / 1e3, 3))
    else:
        fsm = E.fsm_from_priority(wl.priority, len(wl.types))
    staging = E.ED_STAGING_OFF if args.staging == "off" else E.ED_STAGING_AUTO
    step_order = E.ED_ORDER_SCHEDULE if args.step_order == "schedule" else E.ED_ORDER_LEVEL
    plan = E.ed_plan(wl.graphs, wl.types, fsm, layout=layout, staging=staging, step_order=step_order)
    weights = E.DeviceWeights(wl.types, wl.params)
    ws = E.Workspace(plan)
    tdt = torch.bfloat16 if wl.dtype == "bf16" else torch.float32
    rg = None
    if dist:  # the sharded path's one collective (root rows all-gathered over NCCL / NVLink), set up once
        rg = RootGather(wl.shard_idx, wl.n_total, wl.hidden, tdt, "cuda")
        out = rg.local                          # ed_execute writes the roots straight into the send block
    else:
        out = torch.zeros(len(wl.graphs), wl.hidden, dtype=tdt, device="cuda")
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device="cuda")  # 256 MB > L2
    stream = torch.cuda.current_stream()

    for _ in range(args.warmup):
        E.ed_execute(plan, weights, ws, out)
        if rg:
            rg()
    torch.cuda.synchronize()

    clocks = ClockSampler()
    if rank == 0:
        clocks.start()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    step_ns = []
    for k in range(args.steps):
        flush.zero_()                          # untimed: evict L2 between timed steps
        evs[k][0].record(stream)
        E.ed_execute(plan, weights, ws, out)
        if rg:  # the sharded path's one collective: root rows all-gathered (NCCL / NVLink)
            rg()
        evs[k][1].record(stream)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clock_rec = clocks.stop(max(world, 1)) if rank == 0 else None
    times = [a.elapsed_time(b) for a, b in evs]
    ms_local = statistics.median(times)        # median of the timed runs
    step_ns = ws.step_times_ns()               # in-kernel %globaltimer, last timed execute
    ms = ms_local
    if dist:
        t = torch.tensor([ms_local], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    n_inst_total = len(wl.graphs) * world if args.scaling == "weak" else len(W.config(args.config).graphs)
    value = n_inst_total / (ms / 1e3)

    # ---- end to end through the C ABI with host buffers: ed_plan + upload + execute + readback.
    # A serving loop: the minibatch arrives as packed host arrays (GraphBatch, the data loader's
    # output); ed_plan of the next minibatches runs on host threads (PlanPipeline) while the GPU
    # executes the current one; every step uploads its step table + token ids (H2D, inside
    # ed_execute) and reads its instance outputs back into pinned host memory (D2H).
    res_shape = (wl.n_total, wl.hidden) if rg else tuple(out.shape)
    host_out = [torch.empty(res_shape, dtype=out.dtype, pin_memory=True) for _ in range(2)]
    batch = E.GraphBatch(wl.graphs)
    workers = max(1, min(args.plan_threads, (os.cpu_count() or 1) - 2))
    pipe = E.PlanPipeline(wl.types, fsm, workers, layout=layout, staging=staging, step_order=step_order)
    h2d = d2h = 0
    # two workspaces used in turn: the next minibatch's plan is uploaded (H2D + zeroing, on a side
    # stream) into one while the kernel of the current minibatch runs on the other
    wss = [ws, E.Workspace(plan)]
    up_stream = torch.cuda.Stream()

    def e2e_run(nsteps):
        nonlocal h2d, d2h
        window = 2 * workers                                       # minibatches planned ahead (bounded memory)
        futs = [pipe.submit(batch) for _ in range(min(nsteps, window))]
        live = []
        for k in range(nsteps):
            p2 = futs[k].result()                                  # host Alg. 1 + layout + lowering
            futs[k] = None
            if k + window < nsteps:
                futs.append(pipe.submit(batch))
            w_k = wss[k % 2]
            w_k.plan_info = p2.info
            E.ed_execute(p2, weights, w_k, out, upload_stream=up_stream)  # step table H2D on the side stream
            res = rg() if rg else out
            host_out[k % 2].copy_(res, non_blocking=True)          # D2H of the step's result
            h2d, d2h = p2.upload_bytes, host_out[0].numel() * host_out[0].element_size()
            live.append(p2)
            if len(live) > 2:
                live.pop(0)
        torch.cuda.synchronize()

    e2e_run(3)                                                     # warm-up (threads, staging buffers)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    e2e_run(args.e2e_steps)
    b.record(stream)
    torch.cuda.synchronize()
    pipe.close()
    e2e_times = [a.elapsed_time(b) / args.e2e_steps]
    ws.plan_info = plan.info
    for w_ in wss[1:]:
        w_.release()
    e2e_ms = statistics.median(e2e_times)
    if dist:
        t = torch.tensor([e2e_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())

    if rank == 0:
        P, P_sus, BW, src = peaks()
        F_tot, B_tot, troof = plan_roofline(wl, plan, P, BW)
        achieved = F_tot / (ms_local / 1e3) / 1e12
        traffic = None
        prof = os.path.join(ROOT, "profiles", f"ncu_{args.config}_summary.json")
        if os.path.exists(prof):
            traffic = json.load(open(prof)).get("dram_bytes_per_launch")
        meas = [x / 1e9 for x in step_ns]
        t_floor = latency_floor_us(E, wl) if world == 1 or rank == 0 else None
        # device steps -> schedule batches (the kernel walks the batches in dependency-level order,
        # a two-contraction cell has two device steps): t_meas per batch, listed in kernel order
        sched = plan.schedule()
        meas_b = [0.0] * len(sched)
        order = []
        for k, b in enumerate(plan.step_batches()):
            meas_b[b] += meas[k]
            if not order or order[-1] != b:
                order.append(int(b))
        steps_out = [{"batch": b, "type": wl.types[sched[b][0]].name, "m": len(sched[b][1]),
                      "t_roof_us": round(1e6 * troof[b], 3), "t_meas_us": round(1e6 * meas_b[b], 3)} for b in order]
        per_step = {"sum_t_roof_us": 1e6 * sum(troof), "sum_t_meas_us": 1e6 * sum(meas),
                    "frac": (sum(troof) / sum(meas)) if sum(meas) > 0 else None,
                    # secondary: per-step latency floor of the persistent kernel and the
                    # "achievable" fraction sum max(t_roof, t_floor) / sum t_meas
                    "t_floor_us": t_floor,
                    "achievable_frac": (sum(max(1e6 * r, t_floor) for r in troof) / (1e6 * sum(meas)))
                    if (t_floor and sum(meas) > 0) else None,
                    "steps": steps_out}
        cpu_rate, cpu_n, cpu_dt = cpu_oracle_rate(wl, args.cpu_seconds) if world == 1 or rank == 0 else (None, 0, 0)
        all_rate = all_n = all_dt = all_cores = None
        if args.cpu_seconds >= 5 and world == 1:
            try:
                all_rate, all_n, all_dt, all_cores = cpu_oracle_rate_all_cores(args.config, cpu_rate, args.cpu_seconds / 2)
            except Exception as e:  # pragma: no cover - reported, never fatal
                all_rate = f"failed: {e}"
        line = {
            "metric": METRICS[args.config], "value": value, "unit": "instances/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": wl.dtype, "data": "synthetic (seeded parse-like trees, random-init weights)",
            "config": {"workload": CONFIGS[args.config], **fsm_info, "instances_per_gpu": len(wl.graphs),
                       "nodes_per_gpu": wl.num_nodes, "batches": plan.info["num_batches"],
                       "lower_bound": plan.info["lower_bound"], "layout": args.layout, "step_order": args.step_order,
                       "l2": "flushed between timed steps (256 MB write)", "parallelism": f"instance-sharded x{world} ({args.scaling}; LPT by node count when strong)",
                       "split_k_steps": plan.info["split_steps"], "grid": plan.query_info()["grid"]},
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": P, "unit": "TFLOP/s",
                         "frac": achieved / P, "traffic": traffic,
                         "kernel": "ed_persistent_bf16" if wl.dtype == "bf16" else "ed_persistent_f32",
                         "algorithmic_flops_per_launch": F_tot, "algorithmic_bytes_per_launch": B_tot,
                         "peak_source": f"{src} bf16_tflops (burst; kernel timed alone)"},
            "per_step_roofline": per_step,
            # layout evidence (Table 4): what a copy-based executor (DyNet's
            # gather / scatter kernels) would move for this plan's layout, and what the kernel reads as
            # contiguous / staged blocks instead of row gathers
            "layout": {"layout": args.layout, "copy_bytes": plan.info["copy_bytes"],
                       "copy_kernels": plan.info["copy_kernels"], "contig_operands": plan.info["contig_operands"],
                       "gather_operands": plan.info["gather_operands"], "staged_operands": plan.info["staged_operands"],
                       "staged_bytes": plan.info["staged_bytes"], "layout_ms": round(plan.info["layout_us"] / 1e3, 2)},
            "cpu_baseline": {"value": cpu_rate, "unit": "instances/s", "cores": 1, "kind": "oracle",
                             "sample": f"{cpu_n} instances of the {args.config} minibatch in {cpu_dt:.1f} s, fp64 "
                                       "per-node recursive oracle, 1 BLAS thread",
                             "all_cores": {"value": all_rate, "cores": all_cores, "instances": all_n,
                                           "seconds": all_dt, "host": host_cpu()}},
            "e2e": {"value": n_inst_total / (e2e_ms / 1e3), "unit": "instances/s", "ms_per_step": e2e_ms,
                    "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                    "includes": "per step: ed_plan (host Alg. 1 + layout + lowering, on a pool of host threads "
                                "overlapping the GPU) + step-table/token H2D (side stream, two workspaces in turn) + ed_execute + root D2H",
                    "plan_threads": workers},
            "gpu_launches": args.steps * plan.launches,
            "clocks": clock_rec,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
