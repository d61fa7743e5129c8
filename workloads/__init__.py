"""Seeded synthetic workloads for the ED-Batch hot path (harness input only).

This module is shared by the oracle side (tests) and the CUDA side (tests,
bench.py).  It holds NONE of the method's arithmetic: it only draws graph
structures, token ids and parameter values from a counter-based generator and
returns plain numpy arrays.  Every recipe below is stated in DESIGN.md §4
("Input recipe"); the shapes follow SURVEY.md Appendix B and the BASELINE.json
configs.

Graph encoding (one instance = one per-instance dataflow graph, PAPER.md P:73
"dataflow graphs are generated for each of the input instances"):
  type[n]      op-type index of each node (index into Workload.types)
  in_off[n+1]  CSR offsets into in_idx
  in_idx[...]  slot-ordered inputs: >= 0 local node id; ZERO_INPUT = zero state;
               other negatives = external input id (-1 - id), e.g. a word leaf
  ext[n]       token id read by the op from its embedding table, or -1
  root         local node id whose h is the instance output (or -1 - id when the
               instance has no ops and its output is the external row itself)
"""
from __future__ import annotations

import dataclasses
from typing import Dict, List, Optional, Sequence

import numpy as np

ZERO_INPUT = -(2 ** 31)  # INT32_MIN, matches ED_ZERO_INPUT in include/ed_batch.h

MASK64 = (1 << 64) - 1


class SplitMix64:
    """Counter-based SplitMix64 stream (harness RNG)."""

    def __init__(self, seed: int):
        self.state = seed & MASK64

    def next_u64(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & MASK64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        return z ^ (z >> 31)

    def randint(self, lo: int, hi: int) -> int:
        """Uniform integer in [lo, hi] (inclusive)."""
        return lo + self.next_u64() % (hi - lo + 1)

    def uniform01(self) -> float:
        return (self.next_u64() >> 11) * (1.0 / (1 << 53))


@dataclasses.dataclass
class OpType:
    name: str            # short label used in schedules, e.g. "L", "I", "O"
    kind: str            # cell kind, e.g. "treelstm_internal" (see include/ed_batch.h ED_CELL_*)
    num_slots: int       # fixed input slots
    variadic: int = 0    # 1: extra node inputs after the fixed slots (lattice char cell)
    has_ext: int = 0     # 1: reads an embedding row by ext[v]
    weight_set: int = 0  # index into Workload.params
    hidden: int = 0
    out_dim: int = 0     # logits width for output cells
    dtype: str = "bf16"  # "bf16" | "fp32"


@dataclasses.dataclass
class Graph:
    type: np.ndarray
    in_off: np.ndarray
    in_idx: np.ndarray
    ext: np.ndarray
    root: int

    @property
    def num_nodes(self) -> int:
        return int(self.type.shape[0])

    def inputs(self, v: int) -> np.ndarray:
        return self.in_idx[self.in_off[v]:self.in_off[v + 1]]


@dataclasses.dataclass
class Workload:
    name: str
    types: List[OpType]
    graphs: List[Graph]
    priority: List[int]                 # FSM table as a type-priority list (SURVEY A-3/A-8)
    params: List[Dict[str, np.ndarray]]  # one dict per weight set, fp32 values
    dtype: str
    hidden: int
    config: Dict[str, object] = dataclasses.field(default_factory=dict)

    @property
    def num_nodes(self) -> int:
        return sum(g.num_nodes for g in self.graphs)


class _GraphBuilder:
    def __init__(self):
        self.type: List[int] = []
        self.inputs: List[List[int]] = []
        self.ext: List[int] = []

    def add(self, t: int, inputs: Sequence[int], ext: int = -1) -> int:
        self.type.append(t)
        self.inputs.append(list(inputs))
        self.ext.append(ext)
        return len(self.type) - 1

    def build(self, root: int) -> Graph:
        off = np.zeros(len(self.type) + 1, dtype=np.int32)
        for i, ins in enumerate(self.inputs):
            off[i + 1] = off[i] + len(ins)
        flat = [x for ins in self.inputs for x in ins]
        return Graph(type=np.asarray(self.type, dtype=np.int32), in_off=off,
                     in_idx=np.asarray(flat, dtype=np.int32),
                     ext=np.asarray(self.ext, dtype=np.int32), root=int(root))


def graph_from_lists(types: Sequence[int], inputs: Sequence[Sequence[int]],
                     ext: Optional[Sequence[int]] = None, root: int = -1) -> Graph:
    b = _GraphBuilder()
    for i, t in enumerate(types):
        b.add(t, inputs[i], -1 if ext is None else ext[i])
    return b.build(root if root >= 0 else len(types) - 1)


# ----------------------------------------------------------------------------------------------
# Structures
# ----------------------------------------------------------------------------------------------

def tree_graph(n_leaves: int, rng: SplitMix64, tok: SplitMix64, vocab: int,
               t_leaf: Optional[int], t_int: int, t_out: Optional[int], t_int2: Optional[int] = None) -> Graph:
    """Tree(n): uniform split point k ~ U[1, n-1]; nodes numbered in post-order.

    t_leaf is None -> leaves are external lookups (TreeFC / MV-RNN, SURVEY A-6): internal
    nodes reference them as external ids (-1 - word).  t_out not None -> one output op O
    per L/I node, appended after all tree nodes in node order (SURVEY A-7).  t_int2 not None ->
    TreeLSTM-2Type (Table 1): each internal node is t_int or t_int2 with probability 1/2
    (one SplitMix64 draw after its children are built).
    """
    b = _GraphBuilder()

    def build(n: int) -> int:
        if n == 1:
            word = tok.randint(0, vocab - 1)
            if t_leaf is None:
                return -1 - word
            return b.add(t_leaf, [], word)
        k = rng.randint(1, n - 1)
        left = build(k)
        right = build(n - k)
        t = t_int if t_int2 is None or rng.next_u64() % 2 == 0 else t_int2
        return b.add(t, [left, right])

    root = build(n_leaves)
    if t_out is not None:
        for v in range(len(b.type)):
            b.add(t_out, [v])
    return b.build(root)


def bichain_graph(length: int, tok: SplitMix64, vocab: int, t_f: int, t_b: int, t_t: Optional[int]) -> Graph:
    """BiChain(L): forward chain F_0..F_{L-1}, backward chain B_{L-1}..B_0, tagger T_t(F_t, B_t)
    (t_t None: no tagger ops).  The instance output (root) is the final forward state F_{L-1}."""
    b = _GraphBuilder()
    tokens = [tok.randint(0, vocab - 1) for _ in range(length)]
    f_ids, b_ids = [], [None] * length
    prev = ZERO_INPUT
    for t in range(length):
        prev = b.add(t_f, [prev], tokens[t])
        f_ids.append(prev)
    prev = ZERO_INPUT
    for t in range(length - 1, -1, -1):
        prev = b.add(t_b, [prev], tokens[t])
        b_ids[t] = prev
    if t_t is not None:
        for t in range(length):
            b.add(t_t, [f_ids[t], b_ids[t]])
    return b.build(f_ids[-1])


def lattice_graph(n_chars: int, rng: SplitMix64, tok: SplitMix64, char_vocab: int, word_vocab: int,
                  t_char: int, t_word: int, p_word: float = 0.3, word_end_char: bool = True) -> Graph:
    """Lattice(n) (PAPER Fig. 7): char chain plus word skip cells.

    Word W(b->e), e = min(n-1, b+L-1), L ~ U{2,3,4}, added with probability p for b in 0..n-2;
    duplicates dropped.  C_e slots: [C_{e-1} (ZERO for e=0), words ending at e ascending b].
    W slots: [C_b, external char token of e]; nodes numbered C_e then the words starting at e.
    """
    chars = [tok.randint(0, char_vocab - 1) for _ in range(n_chars)]
    words = []
    seen = set()
    for bpos in range(n_chars - 1):
        if rng.uniform01() < p_word:
            span = rng.randint(2, 4)
            e = min(n_chars - 1, bpos + span - 1)
            if (bpos, e) not in seen:
                seen.add((bpos, e))
                words.append((bpos, e))
    word_tok = {w: tok.randint(0, word_vocab - 1) for w in words}
    ends: Dict[int, List[int]] = {}
    bld = _GraphBuilder()
    char_id: List[int] = []
    word_id: Dict[tuple, int] = {}
    for e in range(n_chars):
        slots = [char_id[e - 1] if e > 0 else ZERO_INPUT]
        slots += [word_id[w] for w in sorted(ends.get(e, []))]
        char_id.append(bld.add(t_char, slots, chars[e]))
        for w in words:
            if w[0] == e:
                slots = [char_id[e], -1 - chars[w[1]]] if word_end_char else [char_id[e]]
                word_id[w] = bld.add(t_word, slots, word_tok[w])
                ends.setdefault(w[1], []).append(w)
    return bld.build(char_id[-1])


# ----------------------------------------------------------------------------------------------
# Parameters (SURVEY A-17)
# ----------------------------------------------------------------------------------------------

def round_to_bf16(x: np.ndarray) -> np.ndarray:
    """Round fp32 values to the nearest bf16-representable fp32 (ties to even).

    Input preparation only: the bf16 path stores these values exactly, and the oracle upcasts
    the same values to fp64 (SURVEY §8(c) "the same (bf16-rounded) weights and inputs").
    """
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def _uniform(gen: np.random.Generator, shape, bound: float) -> np.ndarray:
    return gen.uniform(-bound, bound, size=shape).astype(np.float32)


# logical parameter shapes per cell kind: name -> (rows, cols) in units of h (C = out_dim)
def make_params(kind: str, h: int, gen: np.random.Generator, vocab: int = 0, out_dim: int = 0,
                vocab2: int = 0) -> Dict[str, np.ndarray]:
    s = 1.0 / np.sqrt(h)
    p: Dict[str, np.ndarray] = {}
    if kind == "treelstm_leaf":
        p["W"] = _uniform(gen, (3 * h, h), s); p["b"] = _uniform(gen, (3 * h,), s)
        p["emb"] = _uniform(gen, (vocab, h), 1.0)
    elif kind == "treelstm_internal":
        p["W"] = _uniform(gen, (5 * h, 2 * h), s); p["b"] = _uniform(gen, (5 * h,), s)
    elif kind == "linear_out":
        p["W"] = _uniform(gen, (out_dim, h), s); p["b"] = _uniform(gen, (out_dim,), s)
    elif kind == "treegru_leaf":
        p["W"] = _uniform(gen, (2 * h, h), s); p["b"] = _uniform(gen, (2 * h,), s)
        p["emb"] = _uniform(gen, (vocab, h), 1.0)
    elif kind == "treegru_internal":
        # rows: [z; r_l; r_r] over [h_l; h_r], then a_l = U_nl h_l, a_r = U_nr h_r (block zeros)
        W = _uniform(gen, (5 * h, 2 * h), s)
        W[3 * h:4 * h, h:] = 0.0
        W[4 * h:5 * h, :h] = 0.0
        p["W"] = W; p["b"] = _uniform(gen, (5 * h,), s)
    elif kind == "treefc_internal":
        p["W"] = _uniform(gen, (h, 2 * h), s); p["b"] = _uniform(gen, (h,), s)
        p["emb"] = _uniform(gen, (vocab, h), 1.0)
    elif kind == "lstm":
        p["W"] = _uniform(gen, (4 * h, 2 * h), s); p["b"] = _uniform(gen, (4 * h,), s)
        p["emb"] = _uniform(gen, (vocab, h), 1.0)
    elif kind == "tagger":
        p["W"] = _uniform(gen, (h, 2 * h), s); p["b"] = _uniform(gen, (h,), s)
        p["W2"] = _uniform(gen, (out_dim, h), s); p["b2"] = _uniform(gen, (out_dim,), s)
    elif kind == "mvrnn_internal":
        p["W"] = _uniform(gen, (h, 2 * h), s); p["b"] = _uniform(gen, (h,), s)
        eye = np.eye(h, dtype=np.float32)
        p["WM"] = (np.concatenate([eye / 2, eye / 2], axis=1)
                   + _uniform(gen, (h, 2 * h), 0.01)).astype(np.float32)
        p["emb"] = _uniform(gen, (vocab, h), 1.0)
        p["mat"] = (eye[None, :, :] + _uniform(gen, (vocab, h, h), 0.01)).astype(np.float32)
    elif kind == "lattice_char":
        p["W"] = _uniform(gen, (4 * h, 2 * h), s); p["b"] = _uniform(gen, (4 * h,), s)
        p["emb"] = _uniform(gen, (vocab, h), 1.0)
    elif kind in ("latticegru_char", "latticegru_word"):
        # GRUCell weights stacked over [x; h]: rows [r; z; n_x; n_h]; n_x reads x only, n_h h only
        W = _uniform(gen, (4 * h, 2 * h), s)
        W[2 * h:3 * h, h:] = 0.0
        W[3 * h:, :h] = 0.0
        p["W"] = W; p["b"] = _uniform(gen, (4 * h,), s)
        p["emb"] = _uniform(gen, (vocab, h), 1.0)
    elif kind == "lattice_word":
        p["W"] = _uniform(gen, (3 * h, 2 * h), s); p["b"] = _uniform(gen, (3 * h,), s)
        p["Wl"] = _uniform(gen, (h, 2 * h), s); p["bl"] = _uniform(gen, (h,), s)
        p["emb"] = _uniform(gen, (vocab, h), 1.0)      # word table (ext)
        p["emb2"] = _uniform(gen, (vocab2, h), 1.0)    # char table (external slot x_e)
    else:
        raise ValueError(f"unknown cell kind {kind}")
    return p


def _finish_params(params: List[Dict[str, np.ndarray]], dtype: str) -> List[Dict[str, np.ndarray]]:
    """bf16 path: every value the GPU stores in bf16 (weights, tables) is pre-rounded; biases
    stay fp32 (added in the fp32 epilogue)."""
    if dtype != "bf16":
        return params
    out = []
    for p in params:
        q = {}
        for k, v in p.items():
            q[k] = v if k in ("b", "b2", "bl") else round_to_bf16(v)
        out.append(q)
    return out


# ----------------------------------------------------------------------------------------------
# Configurations (BASELINE.json configs; seeds SURVEY §8(d): graphs 1000+cfg, weights 2000+cfg,
# inputs 3000+cfg)
# ----------------------------------------------------------------------------------------------

def treelstm(n_trees: int, leaves: tuple, h: int, dtype: str, cfg: int, vocab: int = 10000,
             out_dim: int = 5, with_output: bool = True, cell: str = "treelstm") -> Workload:
    """TreeLSTM / TreeGRU forests: types L (leaf cell), I (internal cell), O (output linear)."""
    rng = SplitMix64(1000 + cfg)
    tok = SplitMix64(3000 + cfg)
    types = [OpType("L", f"{cell}_leaf", 0, has_ext=1, weight_set=0, hidden=h, dtype=dtype),
             OpType("I", f"{cell}_internal", 2, weight_set=1, hidden=h, dtype=dtype)]
    if with_output:
        types.append(OpType("O", "linear_out", 1, weight_set=2, hidden=h, out_dim=out_dim, dtype=dtype))
    graphs = []
    for _ in range(n_trees):
        n = rng.randint(leaves[0], leaves[1])
        graphs.append(tree_graph(n, rng, tok, vocab, 0, 1, 2 if with_output else None))
    gen = np.random.default_rng(2000 + cfg)
    params = [make_params(f"{cell}_leaf", h, gen, vocab=vocab),
              make_params(f"{cell}_internal", h, gen)]
    if with_output:
        params.append(make_params("linear_out", h, gen, out_dim=out_dim))
    return Workload(name=f"{cell}_h{h}_{dtype}", types=types, graphs=graphs,
                    priority=list(range(len(types))), params=_finish_params(params, dtype),
                    dtype=dtype, hidden=h,
                    config={"instances": n_trees, "leaves": list(leaves), "cfg": cfg})


def treelstm_2type(n_trees: int, leaves: tuple, h: int, dtype: str, cfg: int, vocab: int = 10000,
                   out_dim: int = 5) -> Workload:
    """TreeLSTM-2Type (Table 1): "an extension to TreeLSTM that contains two types of internal
    nodes, each with 50% probability": types L, I1, I2 (same cell, separate weights), O."""
    rng = SplitMix64(1000 + cfg)
    tok = SplitMix64(3000 + cfg)
    types = [OpType("L", "treelstm_leaf", 0, has_ext=1, weight_set=0, hidden=h, dtype=dtype),
             OpType("I1", "treelstm_internal", 2, weight_set=1, hidden=h, dtype=dtype),
             OpType("I2", "treelstm_internal", 2, weight_set=2, hidden=h, dtype=dtype),
             OpType("O", "linear_out", 1, weight_set=3, hidden=h, out_dim=out_dim, dtype=dtype)]
    graphs = [tree_graph(rng.randint(leaves[0], leaves[1]), rng, tok, vocab, 0, 1, 3, t_int2=2)
              for _ in range(n_trees)]
    gen = np.random.default_rng(2000 + cfg)
    params = [make_params("treelstm_leaf", h, gen, vocab=vocab), make_params("treelstm_internal", h, gen),
              make_params("treelstm_internal", h, gen), make_params("linear_out", h, gen, out_dim=out_dim)]
    return Workload(name=f"treelstm2type_h{h}_{dtype}", types=types, graphs=graphs, priority=[0, 1, 2, 3],
                    params=_finish_params(params, dtype), dtype=dtype, hidden=h,
                    config={"instances": n_trees, "leaves": list(leaves), "cfg": cfg})


def treefc(n_trees: int, leaves: tuple, h: int, dtype: str, cfg: int, vocab: int = 1024,
           cell: str = "treefc") -> Workload:
    """TreeFC / MV-RNN forests: a single internal type; leaves are external lookups (A-6)."""
    rng = SplitMix64(1000 + cfg)
    tok = SplitMix64(3000 + cfg)
    types = [OpType("I", f"{cell}_internal", 2, weight_set=0, hidden=h, dtype=dtype)]
    graphs = []
    for _ in range(n_trees):
        n = rng.randint(leaves[0], leaves[1])
        graphs.append(tree_graph(n, rng, tok, vocab, None, 0, None))
    gen = np.random.default_rng(2000 + cfg)
    params = [make_params(f"{cell}_internal", h, gen, vocab=vocab)]
    return Workload(name=f"{cell}_h{h}_{dtype}", types=types, graphs=graphs, priority=[0],
                    params=_finish_params(params, dtype), dtype=dtype, hidden=h,
                    config={"instances": n_trees, "leaves": list(leaves), "cfg": cfg})


def bilstm(n_seqs: int, lengths: tuple, h: int, dtype: str, cfg: int = 2, vocab: int = 10000,
           out_dim: int = 9, with_tagger: bool = True) -> Workload:
    """BiLSTM tagger: types F, B (LSTM cells, separate weights) and T (tagger MLP)."""
    rng = SplitMix64(1000 + cfg)
    tok = SplitMix64(3000 + cfg)
    types = [OpType("F", "lstm", 1, has_ext=1, weight_set=0, hidden=h, dtype=dtype),
             OpType("B", "lstm", 1, has_ext=1, weight_set=1, hidden=h, dtype=dtype),
             OpType("T", "tagger", 2, weight_set=2, hidden=h, out_dim=out_dim, dtype=dtype)]
    graphs = [bichain_graph(rng.randint(lengths[0], lengths[1]), tok, vocab, 0, 1, 2 if with_tagger else None)
              for _ in range(n_seqs)]
    if not with_tagger:
        types = types[:2]
    gen = np.random.default_rng(2000 + cfg)
    params = [make_params("lstm", h, gen, vocab=vocab), make_params("lstm", h, gen, vocab=vocab),
              make_params("tagger", h, gen, out_dim=out_dim)][:len(types)]
    return Workload(name=f"bilstm_h{h}_{dtype}", types=types, graphs=graphs, priority=list(range(len(types))),
                    params=_finish_params(params, dtype), dtype=dtype, hidden=h,
                    config={"instances": n_seqs, "lengths": list(lengths), "cfg": cfg})


def lattice(n_lattices: int, chars: tuple, h: int, dtype: str, cfg: int = 5, char_vocab: int = 4096,
            word_vocab: int = 16384, p_word: float = 0.3, priority=(0, 1), cell: str = "lattice") -> Workload:
    """LatticeLSTM (cell="lattice") or LatticeGRU (cell="latticegru", A-27): types C (char cell,
    variadic word inputs) and W (word cell); same topology (Fig. 7)."""
    rng = SplitMix64(1000 + cfg)
    tok = SplitMix64(3000 + cfg)
    if cell == "latticegru":
        types = [OpType("C", "latticegru_char", 1, variadic=1, has_ext=1, weight_set=0, hidden=h, dtype=dtype),
                 OpType("W", "latticegru_word", 1, has_ext=1, weight_set=1, hidden=h, dtype=dtype)]
        graphs = [lattice_graph(rng.randint(chars[0], chars[1]), rng, tok, char_vocab, word_vocab, 0, 1, p_word,
                                word_end_char=False) for _ in range(n_lattices)]
        gen = np.random.default_rng(2000 + cfg)
        params = [make_params("latticegru_char", h, gen, vocab=char_vocab),
                  make_params("latticegru_word", h, gen, vocab=word_vocab)]
        return Workload(name=f"latticegru_h{h}_{dtype}", types=types, graphs=graphs, priority=list(priority),
                        params=_finish_params(params, dtype), dtype=dtype, hidden=h,
                        config={"instances": n_lattices, "chars": list(chars), "cfg": cfg})
    types = [OpType("C", "lattice_char", 1, variadic=1, has_ext=1, weight_set=0, hidden=h, dtype=dtype),
             OpType("W", "lattice_word", 2, has_ext=1, weight_set=1, hidden=h, dtype=dtype)]
    graphs = [lattice_graph(rng.randint(chars[0], chars[1]), rng, tok, char_vocab, word_vocab, 0, 1, p_word)
              for _ in range(n_lattices)]
    gen = np.random.default_rng(2000 + cfg)
    params = [make_params("lattice_char", h, gen, vocab=char_vocab),
              make_params("lattice_word", h, gen, vocab=word_vocab, vocab2=char_vocab)]
    return Workload(name=f"lattice_h{h}_{dtype}", types=types, graphs=graphs, priority=list(priority),
                    params=_finish_params(params, dtype), dtype=dtype, hidden=h,
                    config={"instances": n_lattices, "chars": list(chars), "cfg": cfg})


def config(name: str) -> Workload:
    """BASELINE.json configs by short name."""
    if name == "cfg1":
        return treelstm(8, (2, 16), 32, "fp32", 1)
    if name == "cfg2":
        return bilstm(64, (10, 50), 256, "bf16", 2)
    if name == "cfg2_fp32":
        return bilstm(64, (10, 50), 256, "fp32", 2)
    if name == "cfg3":
        return treelstm(256, (5, 40), 512, "bf16", 3)
    if name == "cfg3_gru":
        return treelstm(256, (5, 40), 512, "bf16", 3, cell="treegru")
    if name == "cfg3_2type":
        return treelstm_2type(256, (5, 40), 512, "bf16", 3)
    if name == "cfg4_treefc":
        return treefc(1024, (5, 40), 512, "bf16", 4)
    if name == "cfg4_mvrnn":
        return treefc(1024, (5, 40), 512, "bf16", 4, cell="mvrnn")
    if name == "cfg5":
        return lattice(512, (10, 50), 256, "bf16", 5)
    if name == "cfg5_gru":
        return lattice(512, (10, 50), 256, "bf16", 5, cell="latticegru")
    if name == "cfg5_h512":
        return lattice(512, (10, 50), 512, "bf16", 5)
    raise KeyError(name)


# ----------------------------------------------------------------------------------------------
# Paper fixtures (schedule/layout worked examples)
# ----------------------------------------------------------------------------------------------

def fig1_fixture() -> tuple:
    """PAPER Fig. 1 / §2.1 tree with I, O, R types, as read by SPEC S:43.

    Four leaf inputs (external, depth 0); a left spine of 3 internal ops I1..I3 (depths 1,2,3);
    7 output ops O (on the 4 leaf inputs: depth 1, and on I1..I3: depths 2,3,4); a 6-op
    reduction chain R folding the 7 O outputs in the order O(x1..x4), O(I1), O(I2), O(I3).
    Types: 0 = I, 1 = O, 2 = R.  Returns (graph, type names).
    """
    b = _GraphBuilder()
    i1 = b.add(0, [-1, -2])
    i2 = b.add(0, [i1, -3])
    i3 = b.add(0, [i2, -4])
    outs = [b.add(1, [-1 - k]) for k in range(4)]
    outs += [b.add(1, [i]) for i in (i1, i2, i3)]
    r = b.add(2, [outs[0], outs[1]])
    for o in outs[2:]:
        r = b.add(2, [r, o])
    return b.build(r), ["I", "O", "R"]


def b4_fixture() -> tuple:
    """PAPER App. B.4 "we concatenate two tree networks, but the second has the type of
    Internal node and Output Node swapped": the Fig. 1 tree (types 0 = I, 1 = O, 2 = R) followed by
    a second Fig. 1 tree whose spine ops have type O and whose output ops have type I; the second
    tree's first spine op also reads the first tree's root (the concatenation).  Arities differ
    between the two halves, so op types for the C ABI must be variadic.  Returns (graph, names)."""
    b = _GraphBuilder()
    for half in range(2):
        spine_t, out_t = (0, 1) if half == 0 else (1, 0)
        first_in = [-1, -2] if half == 0 else [prev_root, -2]
        i1 = b.add(spine_t, first_in)
        i2 = b.add(spine_t, [i1, -3])
        i3 = b.add(spine_t, [i2, -4])
        outs = [b.add(out_t, [-1 - k]) for k in range(4)]
        outs += [b.add(out_t, [i]) for i in (i1, i2, i3)]
        r = b.add(2, [outs[0], outs[1]])
        for o in outs[2:]:
            r = b.add(2, [r, o])
        prev_root = r
    return b.build(prev_root), ["I", "O", "R"]


def fig3_fixture() -> tuple:
    """PAPER Fig. 3 / §3.1 as a 3-type DAG (SURVEY §8(c) layout pin, A-25).

    Type A produces x1, x2, x3 from external inputs; alpha: x4 <- (x1, x2), x5 <- (x3, x1)
    (B1's operands {x4,x5}, {x1,x3}, {x2,x1}); sigma: x8 <- x3, x6 <- x4, x7 <- x5 (B2).
    Node ids 0..7 are x1..x8.  Types: 0 = A, 1 = alpha, 2 = sigma.
    """
    b = _GraphBuilder()
    x1 = b.add(0, [-1]); x2 = b.add(0, [-2]); x3 = b.add(0, [-3])
    x4 = b.add(1, [x1, x2]); x5 = b.add(1, [x3, x1])
    x6 = b.add(2, [x4]); x7 = b.add(2, [x5]); x8 = b.add(2, [x3])
    assert (x4, x5, x6, x7, x8) == (3, 4, 5, 6, 7)
    return b.build(x8), ["A", "alpha", "sigma"]
