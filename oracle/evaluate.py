"""fp64 evaluators of a minibatch of per-instance graphs — oracle, test infrastructure only.

SURVEY §8(c) "Outputs": batching only reorders independent work (PAPER P:73, P:112 — a batch
executes exactly the frontier nodes), so the numeric result is the plain per-node evaluation
of each instance's DAG in topological order.  Two independent evaluators are provided:

  evaluate_recursive   memoised per-node recursion using oracle.cells (one node at a time)
  evaluate_levels      level-synchronous: all nodes of one (depth, type) group at once with
                       numpy row-batched matrix products (separate code, not oracle.cells)

They must agree to ~1e-12 (tests/test_oracle_numerics.py).  Records per node:
  {"h": vector, "c": vector | None, "y": logits | None, "M": matrix (MV-RNN) | None}
"""
from __future__ import annotations

import sys
from typing import Dict, List, Optional

import numpy as np

from . import cells
from .graph import Merged, topo_depth

ZERO = -(2 ** 31)


def _p(wl, t):
    return wl.params[wl.types[t].weight_set]


def _ext_rec(wl, t: int, slot: int, xid: int) -> dict:
    """Record of an external input id in slot ``slot`` of a type-t op."""
    ot = wl.types[t]
    p = _p(wl, t)
    if ot.kind == "lattice_word" and slot == 1:
        return {"h": np.asarray(p["emb2"][xid], np.float64), "c": None, "y": None, "M": None}
    rec = {"h": np.asarray(p["emb"][xid], np.float64), "c": None, "y": None, "M": None}
    if ot.kind == "mvrnn_internal":
        rec["M"] = np.asarray(p["mat"][xid], np.float64)
    return rec


def _zero_rec(h: int) -> dict:
    return {"h": np.zeros(h), "c": np.zeros(h), "y": None, "M": None}


def eval_node(wl, t: int, ins: List[dict], ext: int) -> dict:
    """Apply the cell of type t to its input records (slot order)."""
    ot = wl.types[t]
    p = _p(wl, t)
    k = ot.kind
    rec = {"h": None, "c": None, "y": None, "M": None}
    if k in ("treelstm_leaf", "treegru_leaf"):
        x = np.asarray(p["emb"][ext], np.float64)
        if k == "treelstm_leaf":
            rec["h"], rec["c"] = cells.treelstm_leaf(p, x)
        else:
            rec["h"] = cells.treegru_leaf(p, x)
    elif k == "treelstm_internal":
        rec["h"], rec["c"] = cells.treelstm_internal(p, ins[0]["h"], ins[0]["c"], ins[1]["h"], ins[1]["c"])
    elif k == "treegru_internal":
        rec["h"] = cells.treegru_internal(p, ins[0]["h"], ins[1]["h"])
    elif k == "linear_out":
        rec["y"] = cells.linear_out(p, ins[0]["h"])
    elif k == "treefc_internal":
        rec["h"] = cells.treefc_internal(p, ins[0]["h"], ins[1]["h"])
    elif k == "mvrnn_internal":
        rec["h"], rec["M"] = cells.mvrnn_internal(p, ins[0]["h"], ins[0]["M"], ins[1]["h"], ins[1]["M"])
    elif k == "lstm":
        x = np.asarray(p["emb"][ext], np.float64)
        rec["h"], rec["c"] = cells.lstm(p, x, ins[0]["h"], ins[0]["c"])
    elif k == "tagger":
        rec["y"] = cells.tagger(p, ins[0]["h"], ins[1]["h"])
    elif k == "lattice_word":
        xw = np.asarray(p["emb"][ext], np.float64)
        rec["c"], rec["l"] = cells.lattice_word(p, xw, ins[0]["h"], ins[0]["c"], ins[1]["h"])
    elif k == "lattice_char":
        x = np.asarray(p["emb"][ext], np.float64)
        words = [(w["c"], w["l"]) for w in ins[1:]]
        rec["h"], rec["c"] = cells.lattice_char(p, x, ins[0]["h"], ins[0]["c"], words)
    elif k == "latticegru_word":
        rec["h"] = cells.latticegru_word(p, np.asarray(p["emb"][ext], np.float64), ins[0]["h"])
    elif k == "latticegru_char":
        x = np.asarray(p["emb"][ext], np.float64)
        rec["h"] = cells.latticegru_char(p, x, ins[0]["h"], [w["h"] for w in ins[1:]])
    else:
        raise ValueError(k)
    return rec


def evaluate_recursive(wl, instances: Optional[List[int]] = None) -> List[Dict[int, dict]]:
    """Per-instance dict local node id -> record, by memoised recursion on each node."""
    sys.setrecursionlimit(max(10000, sys.getrecursionlimit()))
    out = []
    idx = range(len(wl.graphs)) if instances is None else instances
    for gi in idx:
        g = wl.graphs[gi]
        memo: Dict[int, dict] = {}

        def rec_of(v: int) -> dict:
            if v in memo:
                return memo[v]
            t = int(g.type[v])
            ins = []
            for s, x in enumerate(g.in_idx[g.in_off[v]:g.in_off[v + 1]]):
                x = int(x)
                if x >= 0:
                    ins.append(rec_of(x))
                elif x == ZERO:
                    ins.append(_zero_rec(wl.types[t].hidden))
                else:
                    ins.append(_ext_rec(wl, t, s, -1 - x))
            memo[v] = eval_node(wl, t, ins, int(g.ext[v]))
            return memo[v]

        for v in range(g.num_nodes):
            rec_of(v)
        out.append(memo)
    return out


def root_outputs(wl, recs: List[Dict[int, dict]], instances: Optional[List[int]] = None) -> np.ndarray:
    """Instance outputs in instance order: root h, or the external row when
    an instance has no ops (SURVEY App. B edge case)."""
    rows = []
    idx = range(len(wl.graphs)) if instances is None else instances
    for k, gi in enumerate(idx):
        g = wl.graphs[gi]
        r = int(g.root)
        if r >= 0:
            rows.append(recs[k][r]["h"])
        else:
            rows.append(np.asarray(wl.params[wl.types[0].weight_set]["emb"][-1 - r], np.float64))
    return np.stack(rows)


# ----------------------------------------------------------------------------------------------
# Level-synchronous evaluator (independent code path)
# ----------------------------------------------------------------------------------------------

def _sig(x):
    return 1.0 / (1.0 + np.exp(-x))


def evaluate_levels(wl) -> List[Dict[int, dict]]:
    """Evaluate every (depth, type) group of the merged DAG as one row-batched numpy step."""
    m = Merged(wl.graphs, len(wl.types))
    depth = topo_depth(m)
    H: Dict[int, np.ndarray] = {}
    C: Dict[int, np.ndarray] = {}
    Y: Dict[int, np.ndarray] = {}
    Mx: Dict[int, np.ndarray] = {}
    Lk: Dict[int, np.ndarray] = {}
    groups: Dict[tuple, List[int]] = {}
    for v in range(m.n):
        groups.setdefault((depth[v], m.type[v]), []).append(v)

    def rows(vs, slot, kind_src, t):
        """Stack slot inputs of nodes vs: kind_src 'h' | 'c' | 'M'."""
        ot = wl.types[t]
        p = wl.params[ot.weight_set]
        hdim = ot.hidden
        out = []
        for v in vs:
            k, x = m.inputs[v][slot]
            if k == "n":
                src = {"h": H, "c": C, "M": Mx}[kind_src]
                out.append(src[x])
            elif k == "z":
                out.append(np.zeros(hdim))
            else:
                if kind_src == "M":
                    out.append(np.asarray(p["mat"][x], np.float64))
                elif kind_src == "c":
                    out.append(np.zeros(hdim))
                elif ot.kind == "lattice_word" and slot == 1:
                    out.append(np.asarray(p["emb2"][x], np.float64))
                else:
                    out.append(np.asarray(p["emb"][x], np.float64))
        return np.stack(out)

    for (d, t) in sorted(groups):
        vs = groups[(d, t)]
        ot = wl.types[t]
        p = {k: np.asarray(v, np.float64) for k, v in wl.params[ot.weight_set].items() if k != "mat"}
        h = ot.hidden
        k = ot.kind
        X = None
        if ot.has_ext:
            X = np.asarray(wl.params[ot.weight_set]["emb"][[m.ext[v] for v in vs]], np.float64)
        if k in ("treelstm_leaf",):
            Z = X @ p["W"].T + p["b"]
            c = _sig(Z[:, :h]) * np.tanh(Z[:, 2 * h:])
            hh = _sig(Z[:, h:2 * h]) * np.tanh(c)
        elif k == "treegru_leaf":
            Z = X @ p["W"].T + p["b"]
            hh = (1 - _sig(Z[:, :h])) * np.tanh(Z[:, h:]); c = None
        elif k == "treelstm_internal":
            A = np.concatenate([rows(vs, 0, "h", t), rows(vs, 1, "h", t)], axis=1)
            Z = A @ p["W"].T + p["b"]
            c = (_sig(Z[:, :h]) * np.tanh(Z[:, 4 * h:]) + _sig(Z[:, h:2 * h]) * rows(vs, 0, "c", t)
                 + _sig(Z[:, 2 * h:3 * h]) * rows(vs, 1, "c", t))
            hh = _sig(Z[:, 3 * h:4 * h]) * np.tanh(c)
        elif k == "treegru_internal":
            hl, hr = rows(vs, 0, "h", t), rows(vs, 1, "h", t)
            Z = np.concatenate([hl, hr], axis=1) @ p["W"].T + p["b"]   # zero blocks give a_l, a_r
            n = np.tanh(_sig(Z[:, h:2 * h]) * Z[:, 3 * h:4 * h] + _sig(Z[:, 2 * h:3 * h]) * Z[:, 4 * h:])
            z = _sig(Z[:, :h])
            hh = (1 - z) * n + z * (hl + hr); c = None
        elif k == "linear_out":
            Y.update(zip(vs, rows(vs, 0, "h", t) @ p["W"].T + p["b"]))
            continue
        elif k == "treefc_internal":
            hh = np.tanh(np.concatenate([rows(vs, 0, "h", t), rows(vs, 1, "h", t)], axis=1) @ p["W"].T + p["b"])
            c = None
        elif k == "mvrnn_internal":
            a, b = rows(vs, 0, "h", t), rows(vs, 1, "h", t)
            Am, Bm = rows(vs, 0, "M", t), rows(vs, 1, "M", t)
            Ba = np.einsum("nij,nj->ni", Bm, a)
            Ab = np.einsum("nij,nj->ni", Am, b)
            hh = np.tanh(np.concatenate([Ba, Ab], axis=1) @ p["W"].T + p["b"])
            P = np.einsum("ik,nkj->nij", p["WM"], np.concatenate([Am, Bm], axis=1))
            Mx.update(zip(vs, P)); c = None
        elif k == "lstm":
            Z = np.concatenate([X, rows(vs, 0, "h", t)], axis=1) @ p["W"].T + p["b"]
            c = _sig(Z[:, h:2 * h]) * rows(vs, 0, "c", t) + _sig(Z[:, :h]) * np.tanh(Z[:, 2 * h:3 * h])
            hh = _sig(Z[:, 3 * h:]) * np.tanh(c)
        elif k == "tagger":
            T1 = np.tanh(np.concatenate([rows(vs, 0, "h", t), rows(vs, 1, "h", t)], axis=1) @ p["W"].T + p["b"])
            Y.update(zip(vs, T1 @ p["W2"].T + p["b2"]))
            continue
        elif k == "lattice_word":
            Z = np.concatenate([X, rows(vs, 0, "h", t)], axis=1) @ p["W"].T + p["b"]
            cw = _sig(Z[:, h:2 * h]) * rows(vs, 0, "c", t) + _sig(Z[:, :h]) * np.tanh(Z[:, 2 * h:])
            L = _sig(np.concatenate([rows(vs, 1, "h", t), cw], axis=1) @ p["Wl"].T + p["bl"])
            C.update(zip(vs, cw)); Lk.update(zip(vs, L))
            continue
        elif k == "lattice_char":
            Z = np.concatenate([X, rows(vs, 0, "h", t)], axis=1) @ p["W"].T + p["b"]
            si, sf, so, tg = _sig(Z[:, :h]), _sig(Z[:, h:2 * h]), _sig(Z[:, 2 * h:3 * h]), np.tanh(Z[:, 3 * h:])
            cp = rows(vs, 0, "c", t)
            c = np.empty_like(cp)
            for r, v in enumerate(vs):
                ws = [x for kk, x in m.inputs[v][1:] if kk == "n"]
                if not ws:
                    c[r] = sf[r] * cp[r] + si[r] * tg[r]
                else:
                    num_e = np.exp(si[r])
                    den = num_e + sum(np.exp(Lk[w]) for w in ws)
                    c[r] = num_e / den * tg[r] + sum(np.exp(Lk[w]) / den * C[w] for w in ws)
            hh = so * np.tanh(c)
        elif k in ("latticegru_word", "latticegru_char"):
            HP = rows(vs, 0, "h", t)
            Z = np.concatenate([X, HP], axis=1) @ p["W"].T + p["b"]
            r_, z_ = _sig(Z[:, :h]), _sig(Z[:, h:2 * h])
            hh = (1.0 - z_) * np.tanh(Z[:, 2 * h:3 * h] + r_ * Z[:, 3 * h:]) + z_ * HP; c = None
            if k == "latticegru_char":
                for r, v in enumerate(vs):
                    for kk, x in m.inputs[v][1:]:
                        if kk == "n":
                            hh[r] = np.maximum(hh[r], H[x])
        else:
            raise ValueError(k)
        H.update(zip(vs, hh))
        if c is not None:
            C.update(zip(vs, c))

    out = []
    for gi, g in enumerate(wl.graphs):
        base = m.base[gi]
        d = {}
        for v in range(g.num_nodes):
            gv = base + v
            d[v] = {"h": H.get(gv), "c": C.get(gv), "y": Y.get(gv), "M": Mx.get(gv), "l": Lk.get(gv)}
        out.append(d)
    return out
