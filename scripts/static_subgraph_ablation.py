"""Static-subgraph memory-layout ablation (PAPER §3; Table 4).

The paper plans PQ-tree layouts inside each cell's static subgraph (DyNet's unfused op graph of the
cell, parameters included): batching the gate ops needs their operands -- weights among them --
contiguous and aligned, else the executor copies them (gather / scatter kernels).  Here every cell is
one fused kernel, so this is an ablation of the planner only: each cell's op graph (reading S-2 in
DESIGN.md: one plausible DyNet-style decomposition; the paper does not list the ops) at model size 64
(Table 4's setting; counts are per subgraph), batched by Alg. 1 with the DyNet agenda policy through
ed_plan, and the copies a copy-based executor needs are counted for the label (program-order) layout
and for the PQ layout ed_plan returns.  A repeated input (x read by every gate) is a broadcast and is
copied under any layout.  Product API only (ed_plan,
Plan.schedule / layout); the byte count uses each variable's size (a weight is h x h, a vector h).

    python scripts/static_subgraph_ablation.py [--out profiles/static_subgraph_r02]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as W  # noqa: E402
from paper_2302_03851_b200 import edbatch as E  # noqa: E402

H = 64
B = 1  # one cell invocation = one static subgraph (Table 4 counts per subgraph; its batch size 8 only
       # repeats the identical subgraph)
# op kinds -> (cell kind used only for its slot count, slots); planning only, never executed
KINDS = {"param": ("treelstm_leaf", 0), "input": ("treelstm_leaf", 0), "matmul": ("treefc_internal", 2),
         "add": ("treefc_internal", 2), "mul": ("treefc_internal", 2), "sigmoid": ("linear_out", 1),
         "tanh": ("linear_out", 1), "cmult": ("treefc_internal", 2)}
ORDER = list(KINDS)


class Sub:
    """A static subgraph builder: params shared by the B instances, per-instance ops."""

    def __init__(self):
        self.kind, self.ins, self.size = [], [], []

    def node(self, kind, ins, size):
        self.kind.append(kind)
        self.ins.append(list(ins))
        self.size.append(size)
        return len(self.kind) - 1


def lstm_cell(s, P, x, hp, cp):
    g = {}
    for k in "ifou":
        a = s.node("matmul", [P["W" + k], x], H)
        r = s.node("matmul", [P["U" + k], hp], H)
        z = s.node("add", [s.node("add", [a, r], H), P["b" + k]], H)
        g[k] = s.node("tanh" if k == "u" else "sigmoid", [z], H)
    c = s.node("add", [s.node("mul", [g["f"], cp], H), s.node("mul", [g["i"], g["u"]], H)], H)
    return s.node("mul", [g["o"], s.node("tanh", [c], H)], H)


def gru_cell(s, P, x, hp):
    g = {}
    for k in "rz":
        a = s.node("matmul", [P["W" + k], x], H)
        r = s.node("matmul", [P["U" + k], hp], H)
        g[k] = s.node("sigmoid", [s.node("add", [s.node("add", [a, r], H), P["b" + k]], H)], H)
    nx = s.node("add", [s.node("matmul", [P["Wn"], x], H), P["bn"]], H)
    nh = s.node("matmul", [P["Un"], hp], H)
    n = s.node("tanh", [s.node("add", [nx, s.node("mul", [g["r"], nh], H)], H)], H)
    zn = s.node("cmult", [g["z"], n], H)        # (1 - z) n written as one op
    return s.node("add", [zn, s.node("mul", [g["z"], hp], H)], H)


def treelstm_internal(s, P, hl, cl, hr, cr):
    g = {}
    for k in ("i", "fl", "fr", "o", "u"):
        a = s.node("matmul", [P["Ul" + k], hl], H)
        r = s.node("matmul", [P["Ur" + k], hr], H)
        g[k] = s.node("tanh" if k == "u" else "sigmoid", [s.node("add", [s.node("add", [a, r], H), P["b" + k]], H)], H)
    c = s.node("add", [s.node("add", [s.node("mul", [g["fl"], cl], H), s.node("mul", [g["fr"], cr], H)], H),
                       s.node("mul", [g["i"], g["u"]], H)], H)
    return s.node("mul", [g["o"], s.node("tanh", [c], H)], H)


def treelstm_leaf(s, P, x):
    g = {}
    for k in "iou":
        g[k] = s.node("tanh" if k == "u" else "sigmoid", [s.node("add", [s.node("matmul", [P["W" + k], x], H), P["b" + k]], H)], H)
    c = s.node("mul", [g["i"], g["u"]], H)
    return s.node("mul", [g["o"], s.node("tanh", [c], H)], H)


def treegru_internal(s, P, hl, hr):
    g = {}
    for k in ("z", "rl", "rr"):
        g[k] = s.node("sigmoid", [s.node("add", [s.node("add", [s.node("matmul", [P["Ul" + k], hl], H),
                                                               s.node("matmul", [P["Ur" + k], hr], H)], H), P["b" + k]], H)], H)
    al = s.node("add", [s.node("matmul", [P["Unl"], hl], H), P["bnl"]], H)
    ar = s.node("add", [s.node("matmul", [P["Unr"], hr], H), P["bnr"]], H)
    n = s.node("tanh", [s.node("add", [s.node("mul", [g["rl"], al], H), s.node("mul", [g["rr"], ar], H)], H)], H)
    hs = s.node("add", [hl, hr], H)
    return s.node("add", [s.node("cmult", [g["z"], n], H), s.node("mul", [g["z"], hs], H)], H)


def treegru_leaf(s, P, x):
    z = s.node("sigmoid", [s.node("add", [s.node("matmul", [P["Wz"], x], H), P["bz"]], H)], H)
    n = s.node("tanh", [s.node("add", [s.node("matmul", [P["Wn"], x], H), P["bn"]], H)], H)
    return s.node("cmult", [z, n], H)


def mv_cell(s, P, a, A, b, Bm):
    ba = s.node("matmul", [Bm, a], H)
    ab = s.node("matmul", [A, b], H)
    p = s.node("tanh", [s.node("add", [s.node("add", [s.node("matmul", [P["Wl"], ba], H), s.node("matmul", [P["Wr"], ab], H)], H),
                                       P["b"]], H)], H)
    M = s.node("add", [s.node("matmul", [P["WMl"], A], H * H), s.node("matmul", [P["WMr"], Bm], H * H)], H * H)
    return p, M


CELLS = {
    "GRUCell": (["Wr", "Ur", "br", "Wz", "Uz", "bz", "Wn", "bn", "Un"], ["x", "hp"], gru_cell),
    "LSTMCell": ([p + k for k in "ifou" for p in ("W", "U", "b")], ["x", "hp", "cp"], lstm_cell),
    "MVCell": (["Wl", "Wr", "b", "WMl", "WMr"], ["a", "A", "b", "B"], mv_cell),
    "TreeGRU-Internal": ([p + k for k in ("z", "rl", "rr") for p in ("Ul", "Ur", "b")] + ["Unl", "bnl", "Unr", "bnr"],
                         ["hl", "hr"], treegru_internal),
    "TreeGRU-Leaf": (["Wz", "bz", "Wn", "bn"], ["x"], treegru_leaf),
    "TreeLSTM-Internal": ([p + k for k in ("i", "fl", "fr", "o", "u") for p in ("Ul", "Ur", "b")], ["hl", "cl", "hr", "cr"],
                          treelstm_internal),
    "TreeLSTM-Leaf": ([p + k for k in "iou" for p in ("W", "b")], ["x"], treelstm_leaf),
}


def build(name):
    params, inputs, fn = CELLS[name]
    s = Sub()
    P = {p: s.node("param", [], H * H if p[0] in "WU" else H) for p in params}   # shared by the B instances
    for _ in range(B):
        iv = {v: s.node("input", [], H * H if v in ("A", "B") else H) for v in inputs}
        fn(s, P, *[iv[v] for v in inputs])
    return s


def copies(sched, row, s, broadcasts_only=False):
    """Copy kernels / bytes of a copy-based executor: members in result-row order; every operand not
    consecutive-ascending in memory is gathered (sources) or scattered (result): 2 x its bytes."""
    kernels = nbytes = 0
    for t, mem in sched:
        mem = sorted(mem, key=lambda v: row[v])
        ops = [list(mem)]
        for j in range(len(s.ins[mem[0]])):
            src = [s.ins[v][j] for v in mem]
            if len(set(src)) < len(src):           # a repeated input (x shared by the gates) is a
                kernels += 1                       # broadcast: copied whatever the layout
                nbytes += 2 * 4 * sum(s.size[v] for v in src)
            else:
                ops.append(src)
        for op in ([] if broadcasts_only else ops):
            r = [row[v] for v in op]
            if any(r[k + 1] != r[k] + 1 for k in range(len(r) - 1)):
                kernels += 1
                nbytes += 2 * 4 * sum(s.size[v] for v in op)
    return kernels, nbytes


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "static_subgraph_r02"))
    args = ap.parse_args()
    types = [W.OpType(k, KINDS[k][0], KINDS[k][1], weight_set=i, hidden=H,
                      has_ext=1 if KINDS[k][1] == 0 else 0, out_dim=1 if KINDS[k][0] == "linear_out" else 0,
                      dtype="fp32") for i, k in enumerate(ORDER)]
    lines = ["# Static-subgraph layout ablation (PAPER Table 4 P:351-370: per cell subgraph, model size 64)", "",
             "Each cell's op graph (DESIGN.md reading S-2), parameters included, batched by the DyNet agenda policy",
             "through ed_plan; copy kernels / bytes a copy-based executor needs per subgraph, label layout vs",
             "the PQ layout ed_plan plans (`scripts/static_subgraph_ablation.py`).", "",
             "| subgraph | ops | batches | mem kernels label / PQ | ratio | memcpy kB label / PQ | ratio | PQ ideal (only broadcasts left) |",
             "|---|---|---|---|---|---|---|---|"]
    for name in CELLS:
        s = build(name)
        ext = [v if KINDS[s.kind[v]][1] == 0 else -1 for v in range(len(s.kind))]
        g = W.graph_from_lists([ORDER.index(k) for k in s.kind], s.ins, ext, root=len(s.kind) - 1)
        label = E.ed_plan([g], types, [], policy=E.ED_POLICY_AGENDA)
        pq = E.ed_plan([g], types, [], policy=E.ED_POLICY_AGENDA, layout=E.ED_LAYOUT_PQ)
        sched = label.schedule()
        k0, b0 = copies(sched, list(range(len(s.kind))), s)
        k1, b1 = copies(pq.schedule(), list(pq.layout()), s)
        _, bc = copies(pq.schedule(), list(range(len(s.kind))), s, broadcasts_only=True)
        ideal = "yes" if b1 == bc else "no"
        lines.append(f"| {name} | {len(s.kind)} | {len(sched)} | {k0} / {k1} | {k0 / max(k1, 1):.1f} | "
                     f"{b0 / 1e3:.1f} / {b1 / 1e3:.1f} | {b0 / max(b1, 1):.1f} | {ideal} |")
        print(lines[-1], flush=True)
    open(args.out + ".md", "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
