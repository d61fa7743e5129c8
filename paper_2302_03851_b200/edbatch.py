"""Thin ctypes binding of libedbatch.so (include/ed_batch.h) — argument marshalling only.

Every step of the hot path runs in the library: ed_plan (host C++ scheduler + layout planner)
and ed_execute (one persistent sm_100a kernel).  PyTorch supplies device memory and streams.
There is no fallback: if libedbatch.so is missing this module raises at import time.
"""
from __future__ import annotations

import ctypes
import os
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ED_BATCH_LIB") or os.path.join(_HERE, "libedbatch.so")  # override: A/B builds

ED_OK = 0
ED_ZERO_INPUT = -(2 ** 31)
ED_FP32, ED_BF16 = 0, 1
ED_ENC_SORT, ED_ENC_BASE, ED_ENC_MAX = 0, 1, 2
ED_RL_EPISODE_INSTANCE, ED_RL_EPISODE_MERGED = 0, 1
ED_LAYOUT_SCHEDULE_ORDER, ED_LAYOUT_PQ = 0, 1
ED_STAGING_AUTO, ED_STAGING_OFF = 0, 1
ED_POLICY_FSM, ED_POLICY_DEPTH, ED_POLICY_AGENDA, ED_POLICY_SC = 0, 1, 2, 3
ED_ORDER_LEVEL, ED_ORDER_SCHEDULE = 0, 1
STATUS = {0: "ED_OK", -1: "ED_E_INVALID_ARG", -2: "ED_E_CYCLE", -3: "ED_E_DANGLING", -4: "ED_E_DUP_ID",
          -5: "ED_E_TYPE", -6: "ED_E_ARITY", -7: "ED_E_FSM", -8: "ED_E_CUDA", -9: "ED_E_UNSUPPORTED",
          -10: "ED_E_WORKSPACE", -11: "ED_E_OOM"}
CELL = {"treelstm_leaf": 1, "treelstm_internal": 2, "linear_out": 3, "treegru_leaf": 4,
        "treegru_internal": 5, "treefc_internal": 6, "lstm": 7, "tagger": 8, "mvrnn_internal": 9,
        "lattice_char": 10, "lattice_word": 11, "latticegru_char": 12, "latticegru_word": 13}
DTYPE = {"fp32": ED_FP32, "bf16": ED_BF16}

_p = ctypes.POINTER
_i32p = _p(ctypes.c_int32)


class ed_op_type_t(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in
                ("cell_kind", "num_slots", "variadic", "has_ext", "weight_set", "hidden", "out_dim", "dtype")]


class ed_graph_t(ctypes.Structure):
    _fields_ = [("num_nodes", ctypes.c_int32), ("type", _i32p), ("in_off", _i32p), ("in_idx", _i32p),
                ("ext", _i32p), ("root", ctypes.c_int32)]


class ed_fsm_entry_t(ctypes.Structure):
    _fields_ = [("key_len", ctypes.c_int32), ("key", _i32p), ("action", ctypes.c_int32)]


class ed_fsm_t(ctypes.Structure):
    _fields_ = [("encoder", ctypes.c_int32), ("num_entries", ctypes.c_int32), ("entries", _p(ed_fsm_entry_t)),
                ("fallback", ctypes.c_int32)]


class ed_plan_opts_t(ctypes.Structure):
    _fields_ = [("layout", ctypes.c_int32), ("staging", ctypes.c_int32), ("policy", ctypes.c_int32),
                ("step_order", ctypes.c_int32), ("reserved", ctypes.c_int32 * 4)]


_INFO_I64 = ("num_nodes", "num_instances", "num_batches", "num_steps", "lower_bound", "num_rows", "hidden", "dtype",
             "workspace_bytes", "contig_operands", "gather_operands", "copy_bytes", "copy_kernels", "off_h",
             "off_c", "off_y", "y_cols", "off_x", "off_ts", "off_u", "off_m")


class ed_plan_info_t(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in _INFO_I64] + [
        ("plan_us", ctypes.c_double), ("schedule_us", ctypes.c_double), ("layout_us", ctypes.c_double),
        ("staged_operands", ctypes.c_int64), ("staged_bytes", ctypes.c_int64), ("h_rows", ctypes.c_int64),
        ("validate_us", ctypes.c_double), ("lower_us", ctypes.c_double), ("split_steps", ctypes.c_int64),
        ("grid", ctypes.c_int64)]


class ed_weight_set_t(ctypes.Structure):
    _fields_ = [("W", ctypes.c_void_p), ("b", ctypes.c_void_p), ("W2", ctypes.c_void_p), ("b2", ctypes.c_void_p),
                ("emb", ctypes.c_void_p), ("emb2", ctypes.c_void_p), ("mat", ctypes.c_void_p),
                ("emb_rows", ctypes.c_int32), ("emb2_rows", ctypes.c_int32)]


class ed_weights_t(ctypes.Structure):
    _fields_ = [("num_sets", ctypes.c_int32), ("sets", _p(ed_weight_set_t))]


class ed_io_t(ctypes.Structure):
    _fields_ = [("out_root", ctypes.c_void_p), ("trace", ctypes.c_void_p), ("upload_stream", ctypes.c_void_p)]


class ed_rl_config_t(ctypes.Structure):
    _fields_ = [("encoder", ctypes.c_int32), ("n_steps", ctypes.c_int32), ("max_episodes", ctypes.c_int32),
                ("check_every", ctypes.c_int32), ("eps_every", ctypes.c_int32), ("episode_graph", ctypes.c_int32),
                ("alpha", ctypes.c_double), ("lr", ctypes.c_double), ("eps0", ctypes.c_double),
                ("eps_decay", ctypes.c_double), ("eps_floor", ctypes.c_double), ("seed", ctypes.c_uint64)]


class ed_fsm_learned_info_t(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in ("episodes", "table_entries", "q_entries", "checkpoints",
                                               "final_batches", "lower_bound")] + [("learn_us", ctypes.c_double)]


class EdError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code
        self.name = STATUS.get(code, str(code))


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2302_03851_b200.build` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    lib.ed_plan.argtypes = [_p(ed_graph_t), ctypes.c_int32, _p(ed_op_type_t), ctypes.c_int32, _p(ed_fsm_t),
                            _p(ed_plan_opts_t), _p(ctypes.c_void_p)]
    lib.ed_plan_info.argtypes = [ctypes.c_void_p, _p(ed_plan_info_t)]
    lib.ed_plan_get_schedule.argtypes = [ctypes.c_void_p, _i32p, _i32p, _i32p]
    lib.ed_plan_get_layout.argtypes = [ctypes.c_void_p, _i32p]
    lib.ed_plan_get_slot_modes.argtypes = [ctypes.c_void_p, _i32p]
    lib.ed_plan_get_step_batches.argtypes = [ctypes.c_void_p, _i32p]
    lib.ed_plan_destroy.argtypes = [ctypes.c_void_p]
    lib.ed_plan_destroy.restype = None
    lib.ed_packed_bytes.argtypes = [ctypes.c_int32] * 5
    lib.ed_packed_bytes.restype = ctypes.c_int64
    lib.ed_pack_weights.argtypes = [ctypes.c_int32] * 5 + [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
    lib.ed_execute.argtypes = [ctypes.c_void_p, _p(ed_weights_t), _p(ed_io_t), ctypes.c_void_p, ctypes.c_size_t,
                               ctypes.c_void_p]
    lib.ed_execute_launch_count.argtypes = [ctypes.c_void_p]
    if hasattr(lib, "ed_workspace_release") or LIB_PATH.endswith("paper_2302_03851_b200/libedbatch.so"):
        lib.ed_workspace_release.argtypes = [ctypes.c_void_p]  # (older A/B builds via ED_BATCH_LIB lack it)
        lib.ed_workspace_release.restype = ctypes.c_int32
    lib.ed_plan_upload_bytes.argtypes = [ctypes.c_void_p]
    lib.ed_plan_upload_bytes.restype = ctypes.c_int64
    lib.ed_fsm_learn.argtypes = [_p(ed_graph_t), ctypes.c_int32, _p(ed_op_type_t), ctypes.c_int32,
                                 _p(ed_rl_config_t), _p(ctypes.c_void_p)]
    lib.ed_fsm_learned_info.argtypes = [ctypes.c_void_p, _p(ed_fsm_learned_info_t)]
    lib.ed_fsm_learned_table.argtypes = [ctypes.c_void_p, _p(ed_fsm_t)]
    lib.ed_fsm_learned_q.argtypes = [ctypes.c_void_p, ctypes.c_int64, _i32p, _i32p, _i32p, _p(ctypes.c_double)]
    lib.ed_fsm_learned_checkpoint.argtypes = [ctypes.c_void_p, ctypes.c_int64, _p(ctypes.c_int64), _p(ctypes.c_int64)]
    lib.ed_fsm_learned_destroy.argtypes = [ctypes.c_void_p]
    lib.ed_fsm_learned_destroy.restype = None
    for f in ("ed_fsm_learn", "ed_fsm_learned_info", "ed_fsm_learned_table", "ed_fsm_learned_q",
              "ed_fsm_learned_checkpoint"):
        getattr(lib, f).restype = ctypes.c_int32
    lib.ed_last_error.restype = ctypes.c_char_p
    lib.ed_version.restype = ctypes.c_char_p
    for f in ("ed_plan", "ed_plan_info", "ed_plan_get_schedule", "ed_plan_get_layout", "ed_plan_get_slot_modes",
              "ed_plan_get_step_batches",
              "ed_pack_weights", "ed_execute", "ed_execute_launch_count"):
        getattr(lib, f).restype = ctypes.c_int32
    return lib


LIB = _load()


def _check(code: int):
    if code != ED_OK:
        raise EdError(code, LIB.ed_last_error().decode())


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_i32p)


def fsm_from_priority(priority: Sequence[int], num_types: int) -> List[Tuple[Tuple[int, ...], int]]:
    """FSM table as (E_sort key, action) entries for every key: the highest-priority type present."""
    import itertools
    rank = {t: i for i, t in enumerate(priority)}
    out = []
    for k in range(1, num_types + 1):
        for key in itertools.permutations(range(num_types), k):
            out.append((key, min(key, key=lambda t: rank.get(t, len(rank) + t))))
    return out


# ed_graph_t as a numpy record (x86-64 layout: int32, pad, 4 pointers, int32, pad = 48 bytes), so
# that a minibatch of thousands of graphs is marshalled with a few vectorized numpy operations
_GRAPH_REC = np.dtype([("num_nodes", np.int32), ("_p0", np.int32), ("type", np.uint64), ("in_off", np.uint64),
                       ("in_idx", np.uint64), ("ext", np.uint64), ("root", np.int32), ("_p1", np.int32)])
assert _GRAPH_REC.itemsize == ctypes.sizeof(ed_graph_t)


def _graph_arrays(graphs, keep):
    """ed_graph_t[len(graphs)] pointing into four concatenated int32 arrays (kept alive in keep)."""
    n = len(graphs)
    sizes = np.fromiter((len(g.type) for g in graphs), dtype=np.int64, count=n)
    nin = np.fromiter((len(g.in_idx) for g in graphs), dtype=np.int64, count=n)
    cat = lambda xs: np.ascontiguousarray(np.concatenate(xs).astype(np.int32, copy=False)) if n else np.zeros(1, np.int32)
    types = cat([g.type for g in graphs])
    offs = cat([g.in_off for g in graphs])
    idx = cat([g.in_idx for g in graphs] + [np.zeros(1, np.int32)])
    ext = cat([g.ext for g in graphs])
    keep.append((types, offs, idx, ext))
    node_off = np.concatenate([[0], np.cumsum(sizes)[:-1]]) if n else np.zeros(0, np.int64)
    in_off_off = node_off + np.arange(n)                   # each in_off has num_nodes + 1 entries
    idx_off = np.concatenate([[0], np.cumsum(nin)[:-1]]) if n else np.zeros(0, np.int64)
    rec = np.zeros(max(n, 1), dtype=_GRAPH_REC)
    rec["num_nodes"][:n] = sizes
    rec["type"][:n] = types.ctypes.data + 4 * node_off
    rec["in_off"][:n] = offs.ctypes.data + 4 * in_off_off
    rec["in_idx"][:n] = idx.ctypes.data + 4 * idx_off
    rec["ext"][:n] = ext.ctypes.data + 4 * node_off
    rec["root"][:n] = np.fromiter((int(g.root) for g in graphs), dtype=np.int32, count=n)
    keep.append(rec)
    return rec.ctypes.data_as(_p(ed_graph_t))


def _type_array(types):
    tarr = (ed_op_type_t * len(types))()
    for k, t in enumerate(types):
        tarr[k] = ed_op_type_t(CELL[t.kind], t.num_slots, t.variadic, t.has_ext, t.weight_set, t.hidden,
                               t.out_dim, DTYPE[t.dtype])
    return tarr


class LearnedFsm:
    """FSM table learned by ed_fsm_learn (PAPER §2.3): table entries as (key, action), Q values,
    checkpoints (episode, greedy batch total) and info."""

    def __init__(self, handle, num_types: int):
        self.handle = handle
        info = ed_fsm_learned_info_t()
        _check(LIB.ed_fsm_learned_info(handle, ctypes.byref(info)))
        self.info = {n: getattr(info, n) for n, _ in ed_fsm_learned_info_t._fields_}
        f = ed_fsm_t()
        _check(LIB.ed_fsm_learned_table(handle, ctypes.byref(f)))
        self.encoder = f.encoder
        self.table = [(tuple(f.entries[e].key[i] for i in range(f.entries[e].key_len)), f.entries[e].action)
                      for e in range(f.num_entries)]
        self.q = {}
        key = (ctypes.c_int32 * (num_types + 1))()   # E_max keys: type set + argmax type
        kl, a, v = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_double()
        for k in range(self.info["q_entries"]):
            _check(LIB.ed_fsm_learned_q(handle, k, key, ctypes.byref(kl), ctypes.byref(a), ctypes.byref(v)))
            self.q[(tuple(key[i] for i in range(kl.value)), a.value)] = v.value
        self.checkpoints = []
        ep, nb = ctypes.c_int64(), ctypes.c_int64()
        for c in range(self.info["checkpoints"]):
            _check(LIB.ed_fsm_learned_checkpoint(handle, c, ctypes.byref(ep), ctypes.byref(nb)))
            self.checkpoints.append((ep.value, nb.value))

    def __del__(self):
        if getattr(self, "handle", None) and LIB is not None:
            LIB.ed_fsm_learned_destroy(self.handle)
            self.handle = None


def ed_fsm_learn(graphs, types, encoder: int = ED_ENC_SORT, alpha: float = 0.5, lr: float = 0.1, eps0: float = 0.5,
                 eps_decay: float = 0.95, eps_every: int = 10, eps_floor: float = 0.02, n_steps: int = 4,
                 max_episodes: int = 1000, check_every: int = 50, seed: int = 4000,
                 merged: bool = False) -> LearnedFsm:
    """Learn an FSM table by tabular N-step Q-learning (include/ed_batch.h ed_fsm_learn).  merged=True
    runs every episode over the merged minibatch (ED_RL_EPISODE_MERGED) instead of one instance."""
    keep = []
    garr = _graph_arrays(graphs, keep)
    tarr = _type_array(types)
    cfg = ed_rl_config_t(encoder, n_steps, max_episodes, check_every, eps_every,
                         ED_RL_EPISODE_MERGED if merged else ED_RL_EPISODE_INSTANCE, alpha, lr, eps0, eps_decay,
                         eps_floor, seed)
    h = ctypes.c_void_p()
    _check(LIB.ed_fsm_learn(garr, len(graphs), tarr, len(types), ctypes.byref(cfg), ctypes.byref(h)))
    return LearnedFsm(h, len(types))


class Plan:
    """Owning wrapper of an ed_plan_t handle."""

    def __init__(self, handle: ctypes.c_void_p, num_types: int):
        self.handle = handle
        self.num_types = num_types
        info = ed_plan_info_t()
        _check(LIB.ed_plan_info(handle, ctypes.byref(info)))
        self.info = {n: getattr(info, n) for n, _ in ed_plan_info_t._fields_}

    def query_info(self) -> dict:
        """ed_plan_info now (grid is set by the first ed_execute)."""
        info = ed_plan_info_t()
        _check(LIB.ed_plan_info(self.handle, ctypes.byref(info)))
        return {n: getattr(info, n) for n, _ in ed_plan_info_t._fields_}

    def __del__(self):
        if getattr(self, "handle", None) and LIB is not None:
            LIB.ed_plan_destroy(self.handle)
            self.handle = None

    def schedule(self) -> List[Tuple[int, List[int]]]:
        nb, V = self.info["num_batches"], self.info["num_nodes"]
        bt = np.zeros(nb, np.int32); bo = np.zeros(nb + 1, np.int32); mem = np.zeros(max(V, 1), np.int32)
        _check(LIB.ed_plan_get_schedule(self.handle, _ptr(bt), _ptr(bo), _ptr(mem)))
        return [(int(bt[b]), [int(x) for x in mem[bo[b]:bo[b + 1]]]) for b in range(nb)]

    def layout(self) -> np.ndarray:
        row = np.zeros(max(self.info["num_nodes"], 1), np.int32)
        _check(LIB.ed_plan_get_layout(self.handle, _ptr(row)))
        return row[:self.info["num_nodes"]]

    def slot_modes(self) -> np.ndarray:
        m = np.zeros(max(2 * self.info["num_batches"], 1), np.int32)
        _check(LIB.ed_plan_get_slot_modes(self.handle, _ptr(m)))
        return m[:2 * self.info["num_batches"]].reshape(-1, 2)

    def step_batches(self) -> np.ndarray:
        """Schedule batch of every device step, in kernel order (ed_plan_get_step_batches)."""
        sb = np.zeros(max(self.info["num_steps"], 1), np.int32)
        _check(LIB.ed_plan_get_step_batches(self.handle, _ptr(sb)))
        return sb[:self.info["num_steps"]]

    @property
    def upload_bytes(self) -> int:
        return int(LIB.ed_plan_upload_bytes(self.handle))

    @property
    def launches(self) -> int:
        return LIB.ed_execute_launch_count(self.handle)


class GraphBatch:
    """A minibatch of instance graphs packed once into the C ABI's layout (four concatenated int32
    CSR arrays + the ed_graph_t records pointing into them): what a data loader hands to ed_plan.
    Immutable; ed_plan on a GraphBatch does no per-call marshalling of the graphs."""

    def __init__(self, graphs):
        self._keep = []
        self.num_graphs = len(graphs)
        self.garr = _graph_arrays(graphs, self._keep)


def ed_plan(graphs, types, fsm: Sequence[Tuple[Sequence[int], int]], encoder: int = ED_ENC_SORT,
            layout: int = ED_LAYOUT_SCHEDULE_ORDER, staging: int = 0, policy: int = 0,
            step_order: int = 0) -> Plan:
    """graphs: a GraphBatch, or objects with numpy fields type/in_off/in_idx/ext and int root
    (workloads.Graph); types: objects with kind/num_slots/variadic/has_ext/weight_set/hidden/out_dim/dtype.
    The C call runs without the GIL (ctypes), so several host threads can plan concurrently."""
    keep = []
    if isinstance(graphs, GraphBatch):
        garr, ngraphs = graphs.garr, graphs.num_graphs
        keep.append(graphs)
    else:
        garr, ngraphs = _graph_arrays(graphs, keep), len(graphs)
    tarr = _type_array(types)
    earr = (ed_fsm_entry_t * max(len(fsm), 1))()
    for k, (key, act) in enumerate(fsm):
        ka = _i32(list(key))
        keep.append(ka)
        earr[k] = ed_fsm_entry_t(len(ka), _ptr(ka), int(act))
    f = ed_fsm_t(encoder, len(fsm), earr, 0)
    opts = ed_plan_opts_t(layout, staging, policy, step_order, (ctypes.c_int32 * 4)())
    h = ctypes.c_void_p()
    _check(LIB.ed_plan(garr, ngraphs, tarr, len(types), ctypes.byref(f), ctypes.byref(opts), ctypes.byref(h)))
    return Plan(h, len(types))


class PlanPipeline:
    """Plans upcoming minibatches on host threads while the GPU executes the current one (the
    paper's construction + scheduling time, Fig. 6, taken off the critical path of a serving loop).
    submit(batch) -> concurrent.futures.Future[Plan]; results are consumed in submission order by the
    caller, which executes them on its stream.  ed_plan holds no global state, so plans of different
    minibatches are independent."""

    def __init__(self, types, fsm, workers: int, **plan_kw):
        import concurrent.futures as cf
        self.types, self.fsm, self.plan_kw = types, fsm, plan_kw
        self.pool = cf.ThreadPoolExecutor(max_workers=max(1, workers))

    def submit(self, batch):
        return self.pool.submit(ed_plan, batch, self.types, self.fsm, **self.plan_kw)

    def close(self):
        self.pool.shutdown(wait=True)


def _stream_handle(stream) -> ctypes.c_void_p:
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def ed_packed_bytes(kind: str, hidden: int, out_dim: int, dtype: str, which: int) -> int:
    return int(LIB.ed_packed_bytes(CELL[kind], hidden, out_dim, DTYPE[dtype], which))


def ed_pack_weights(kind: str, hidden: int, out_dim: int, dtype: str, which: int, logical: torch.Tensor,
                    stream=None) -> torch.Tensor:
    logical = logical.to(torch.float32).contiguous()
    nbytes = ed_packed_bytes(kind, hidden, out_dim, dtype, which)
    out = torch.empty(nbytes, dtype=torch.uint8, device=logical.device)
    _check(LIB.ed_pack_weights(CELL[kind], hidden, out_dim, DTYPE[dtype], which,
                               ctypes.c_void_p(logical.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                               _stream_handle(stream)))
    return out


_SECOND = {"tagger": ("W2", "b2"), "lattice_word": ("Wl", "bl"), "mvrnn_internal": ("WM", None)}


class DeviceWeights:
    """Weights of a workload on the device, packed by ed_pack_weights (marshalling only)."""

    def __init__(self, types, params: List[Dict[str, np.ndarray]], device="cuda", stream=None):
        self.tensors: List[Dict[str, torch.Tensor]] = []
        tdt = {"bf16": torch.bfloat16, "fp32": torch.float32}
        kinds = {}
        for t in types:
            kinds.setdefault(t.weight_set, t)
        for ws, p in enumerate(params):
            t = kinds.get(ws)
            d: Dict[str, torch.Tensor] = {}
            if t is not None:
                dt = tdt[t.dtype]
                d["W"] = ed_pack_weights(t.kind, t.hidden, t.out_dim, t.dtype, 0,
                                         torch.from_numpy(p["W"]).to(device), stream)
                d["b"] = torch.from_numpy(np.asarray(p["b"], np.float32)).to(device)
                if t.kind in _SECOND:
                    wk, bk = _SECOND[t.kind]
                    d["W2"] = ed_pack_weights(t.kind, t.hidden, t.out_dim, t.dtype, 1,
                                              torch.from_numpy(p[wk]).to(device), stream)
                    if bk:
                        d["b2"] = torch.from_numpy(np.asarray(p[bk], np.float32)).to(device)
                if "mat" in p:  # MV-RNN word matrices: packed (transposed) by the library
                    mat = np.asarray(p["mat"], np.float32)
                    d["mat"] = ed_pack_weights(t.kind, t.hidden, mat.shape[0], t.dtype, 2,
                                               torch.from_numpy(mat).to(device), stream)
                for k in ("emb", "emb2"):
                    if k in p:
                        d[k] = torch.from_numpy(np.asarray(p[k], np.float32)).to(device=device, dtype=dt).contiguous()
            self.tensors.append(d)
        arr = (ed_weight_set_t * len(self.tensors))()
        for k, d in enumerate(self.tensors):
            g = lambda n: ctypes.c_void_p(d[n].data_ptr()) if n in d else None
            arr[k] = ed_weight_set_t(g("W"), g("b"), g("W2"), g("b2"), g("emb"), g("emb2"), g("mat"),
                                     int(d["emb"].shape[0]) if "emb" in d else 0,
                                     int(d["emb2"].shape[0]) if "emb2" in d else 0)
        self._arr = arr
        self.struct = ed_weights_t(len(self.tensors), arr)


class Workspace:
    """Caller-owned device workspace (1024-aligned) with typed views of the row buffers."""

    def __init__(self, plan: Plan, device="cuda"):
        nbytes = int(plan.info["workspace_bytes"])
        self.raw = torch.zeros(nbytes + 1024, dtype=torch.uint8, device=device)
        off = (-self.raw.data_ptr()) % 1024
        self.buf = self.raw[off:off + nbytes]
        self.nbytes = nbytes
        self.plan_info = plan.info

    def release(self) -> None:
        """Unbind the workspace from its plan (ed_workspace_release) and drop the memory: the next
        allocation at this address must not inherit the binding."""
        if getattr(self, "buf", None) is not None:
            if hasattr(LIB, "ed_workspace_release"):
                LIB.ed_workspace_release(ctypes.c_void_p(self.buf.data_ptr()))
            self.buf = None
            self.raw = None

    def __del__(self):
        try:
            self.release()
        except Exception:
            pass

    @property
    def ptr(self) -> int:
        return self.buf.data_ptr()

    def _view(self, off: int, count: int, dtype) -> torch.Tensor:
        es = torch.tensor([], dtype=dtype).element_size()
        return self.buf[off:off + count * es].view(dtype)

    def H(self) -> torch.Tensor:
        i = self.plan_info
        dt = torch.bfloat16 if i["dtype"] == ED_BF16 else torch.float32
        return self._view(i["off_h"], i["num_rows"] * i["hidden"], dt).view(i["num_rows"], i["hidden"])

    def C(self) -> torch.Tensor:
        i = self.plan_info
        return self._view(i["off_c"], i["num_rows"] * i["hidden"], torch.float32).view(i["num_rows"], i["hidden"])

    def Y(self) -> torch.Tensor:
        i = self.plan_info
        return self._view(i["off_y"], i["num_rows"] * i["y_cols"], torch.float32).view(i["num_rows"], i["y_cols"])

    def X(self) -> Optional[torch.Tensor]:
        i = self.plan_info
        if i["off_x"] < 0:
            return None
        return self._view(i["off_x"], i["num_rows"] * i["hidden"], torch.float32).view(i["num_rows"], i["hidden"])

    def U(self) -> Optional[torch.Tensor]:
        """MV-RNN matvec rows [num_rows, 2h] = [B a; A b] (None without MV-RNN types)."""
        i = self.plan_info
        if i["off_u"] < 0:
            return None
        dt = torch.bfloat16 if i["dtype"] == ED_BF16 else torch.float32
        return self._view(i["off_u"], i["num_rows"] * 2 * i["hidden"], dt).view(i["num_rows"], 2 * i["hidden"])

    def M(self) -> Optional[torch.Tensor]:
        """MV-RNN node matrices [num_rows, h, h], each stored transposed (M[r] = P_r^T)."""
        i = self.plan_info
        if i["off_m"] < 0:
            return None
        dt = torch.bfloat16 if i["dtype"] == ED_BF16 else torch.float32
        h = i["hidden"]
        return self._view(i["off_m"], i["num_rows"] * h * h, dt).view(i["num_rows"], h, h)

    def step_times_ns(self) -> np.ndarray:
        """Per device step: time from the completion of all earlier steps to this step's completion
        (stamps are per-step completion maxima; steps overlap in the dataflow kernel, so a step
        finishing before an earlier one gets 0)."""
        i = self.plan_info
        ts = self._view(i["off_ts"], i["num_steps"] + 1, torch.int64).cpu().numpy().astype(np.int64)
        run = np.maximum.accumulate(ts)
        return np.maximum(ts[1:] - run[:-1], 0)


def ed_execute(plan: Plan, weights: DeviceWeights, workspace: Workspace, out_root: Optional[torch.Tensor] = None,
               stream=None, trace: Optional[torch.Tensor] = None, upload_stream=None) -> None:
    info = plan.info
    if out_root is not None:
        want = torch.bfloat16 if info["dtype"] == ED_BF16 else torch.float32
        if not (out_root.is_cuda and out_root.is_contiguous() and out_root.dtype == want
                and out_root.numel() >= info["num_instances"] * info["hidden"]):
            raise ValueError(f"out_root must be a contiguous CUDA {want} tensor with >= "
                             f"{info['num_instances']} x {info['hidden']} elements")
    if trace is not None and not (trace.is_cuda and trace.is_contiguous() and trace.dtype == torch.int64
                                  and trace.numel() >= info["num_steps"] * 64 + 148 * 4):
        raise ValueError("trace must be a contiguous CUDA int64 tensor of >= num_steps * 64 + 148 * 4 elements")
    io = ed_io_t(ctypes.c_void_p(out_root.data_ptr()) if out_root is not None else None,
                 ctypes.c_void_p(trace.data_ptr()) if trace is not None else None,
                 ctypes.c_void_p(upload_stream.cuda_stream) if upload_stream is not None else None)
    _check(LIB.ed_execute(plan.handle, ctypes.byref(weights.struct), ctypes.byref(io),
                          ctypes.c_void_p(workspace.ptr), workspace.nbytes, _stream_handle(stream)))


def version() -> str:
    return LIB.ed_version().decode()
