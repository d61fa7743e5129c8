"""PQ-tree layout planner — oracle, test infrastructure only.

Follows PAPER §3.2 and App. C step by step with the readings of DESIGN.md
§3 (SURVEY A-9..A-13): PQ tree over the node-output variables (Booth–Lueker Reduce, P:180-181,
P:644); results reduced first, then each batch's source operands transactionally in schedule
order; BroadcastConstraint (Alg. 2 / Alg. 3) as forward sweeps until a sweep changes nothing;
canonical form; ParseEquivNodeOrderPair + extended union-find (Alg. 4, Alg. 5) per batch,
transactionally; GetLeafOrder (Alg. 6).

Written independently of the C++ planner: object nodes, pertinence from Python leaf sets, whole-
tree deep copies for transactions.  Parity status: Reduce is pinned by brute force (frontier ==
set of permutations keeping every accepted set consecutive, n <= 7); the whole planner by the
paper's Fig. 3 order, chain closed forms and the plain ideal-layout check; the canonical choice
among equally good layouts is pinned only by bit-exact agreement with the C++ planner
("parity unpinned" beyond that).
"""
from __future__ import annotations

import copy
import itertools
from typing import Dict, List, Optional, Sequence, Tuple

from .graph import Merged

MAX_SWEEPS = 200


class PQNode:
    __slots__ = ("kind", "children", "leaf")

    def __init__(self, kind: str, children=None, leaf: int = -1):
        self.kind = kind            # 'L' leaf, 'P', 'Q'
        self.children: List["PQNode"] = list(children or [])
        self.leaf = leaf

    def leafset(self) -> frozenset:
        if self.kind == "L":
            return frozenset([self.leaf])
        s = set()
        for c in self.children:
            s |= self.leafset_of(c)
        return frozenset(s)

    @staticmethod
    def leafset_of(n) -> frozenset:
        return n.leafset()

    def frontier(self) -> List[int]:
        if self.kind == "L":
            return [self.leaf]
        out = []
        for c in self.children:
            out += c.frontier()
        return out

    def signature(self):
        if self.kind == "L":
            return self.leaf
        return (self.kind, tuple(c.signature() for c in self.children))


class Fail(Exception):
    pass


def _group(kind: str, nodes: List[PQNode]) -> PQNode:
    return nodes[0] if len(nodes) == 1 else PQNode(kind, nodes)


def _normalize(n: PQNode) -> PQNode:
    """1-child nodes collapse; 2-child Q-nodes become P-nodes (standard Booth–Lueker form)."""
    if n.kind == "L":
        return n
    n.children = [_normalize(c) for c in n.children]
    if len(n.children) == 1:
        return n.children[0]
    if n.kind == "Q" and len(n.children) == 2:
        n.kind = "P"
    return n


class PQTree:
    def __init__(self, universe: Sequence[int]):
        leaves = [PQNode("L", leaf=v) for v in universe]
        self.root: Optional[PQNode] = leaves[0] if len(leaves) == 1 else (PQNode("P", leaves) if leaves else None)

    def frontier(self) -> List[int]:
        return self.root.frontier() if self.root is not None else []

    # --- Reduce -----------------------------------------------------------------------------
    def reduce(self, S) -> None:
        """Restrict to orders with S consecutive; raises Fail if impossible (tree then invalid)."""
        S = frozenset(S)
        if len(S) <= 1:
            return
        # pertinent root: deepest node whose leaves contain S
        node, parent = self.root, None
        while True:
            nxt = None
            for c in node.children:
                if S <= c.leafset():
                    nxt = c
                    break
            if nxt is None:
                break
            parent, node = node, nxt
        new = self._reduce_at(node, S, root=True)
        if parent is None:
            self.root = new
        else:
            parent.children = [new if c is node else c for c in parent.children]
        self.root = _normalize(self.root)

    def _label(self, n: PQNode, S) -> str:
        ls = n.leafset()
        if ls <= S:
            return "F"
        if not (ls & S):
            return "E"
        return "P"

    def _reduce_at(self, x: PQNode, S, root: bool) -> PQNode:
        """Returns the replacement of x.  Non-root partial results are Q-nodes ordered
        [empty side ..., full side ...]."""
        if x.kind == "L" or x.leafset() <= S:
            return x
        kids = [c if self._label(c, S) != "P" else self._reduce_at(c, S, False) for c in x.children]
        lab = [self._label(c, S) for c in kids]
        E = [c for c, l in zip(kids, lab) if l == "E"]
        F = [c for c, l in zip(kids, lab) if l == "F"]
        Pt = [c for c, l in zip(kids, lab) if l == "P"]
        if x.kind == "P":
            if not root:
                if not Pt:                                            # template P3
                    return PQNode("Q", [_group("P", E), _group("P", F)])
                if len(Pt) == 1:                                      # template P5
                    seq = ([_group("P", E)] if E else []) + Pt[0].children + ([_group("P", F)] if F else [])
                    return PQNode("Q", seq)
                raise Fail()
            if not Pt:                                                # template P2
                if len(F) >= 2 and E:
                    return PQNode("P", E + [PQNode("P", F)])
                return PQNode("P", kids)
            if len(Pt) == 1:                                          # template P4
                y = PQNode("Q", Pt[0].children + ([_group("P", F)] if F else []))
                return y if not E else PQNode("P", E + [y])
            if len(Pt) == 2:                                          # template P6
                z = PQNode("Q", Pt[0].children + ([_group("P", F)] if F else []) + Pt[1].children[::-1])
                return z if not E else PQNode("P", E + [z])
            raise Fail()
        # Q-node
        if not root:                                                  # template Q2
            for seq_k, seq_l in ((kids, lab), (kids[::-1], lab[::-1])):
                i = 0
                while i < len(seq_l) and seq_l[i] == "E":
                    i += 1
                if i < len(seq_l) and seq_l[i] == "P":
                    i += 1
                while i < len(seq_l) and seq_l[i] == "F":
                    i += 1
                if i == len(seq_l):
                    out = []
                    for c, l in zip(seq_k, seq_l):
                        out += c.children if l == "P" else [c]
                    return PQNode("Q", out)
            raise Fail()
        idx = [i for i, l in enumerate(lab) if l != "E"]             # template Q3
        a, b = idx[0], idx[-1]
        if any(lab[i] == "E" for i in range(a, b + 1)):
            raise Fail()
        if any(lab[i] == "P" and i not in (a, b) for i in range(a, b + 1)) or (a == b):
            raise Fail()
        out = []
        for i, (c, l) in enumerate(zip(kids, lab)):
            if l == "P":
                out += c.children if i == a else c.children[::-1]
            else:
                out.append(c)
        return PQNode("Q", out)

    # --- queries ------------------------------------------------------------------------------
    def min_subtree(self, O) -> Tuple[PQNode, Optional[Tuple[int, int]]]:
        """(node, run): the deepest node holding all of O; run = (first, last) covered children
        when O covers only a run of a Q-node's children, else None."""
        O = frozenset(O)
        node = self.root
        while True:
            nxt = None
            for c in node.children:
                if O <= c.leafset():
                    nxt = c
                    break
            if nxt is None:
                break
            node = nxt
        if node.kind == "L":
            return node, None
        cov = [i for i, c in enumerate(node.children) if c.leafset() & O]
        if cov[0] == 0 and cov[-1] == len(node.children) - 1:
            return node, None
        return node, (cov[0], cov[-1])

    def all_frontiers(self) -> set:
        """Every leaf order the tree allows (P: all permutations, Q: both directions)."""
        def gen(n):
            if n.kind == "L":
                return [[n.leaf]]
            subs = [gen(c) for c in n.children]
            outs = []
            orders = itertools.permutations(range(len(subs))) if n.kind == "P" else \
                [tuple(range(len(subs))), tuple(range(len(subs) - 1, -1, -1))]
            for perm in orders:
                for combo in itertools.product(*[subs[i] for i in perm]):
                    outs.append(sum(combo, []))
            return outs
        return set(tuple(f) for f in gen(self.root))


# ------------------------------------------------------------------------------------------------
# planner
# ------------------------------------------------------------------------------------------------

def batch_operands(m: Merged, sched, fixed_slots: Sequence[int]) -> List[List[List[int]]]:
    """Per batch: [result (members ascending id), constrained source operands aligned by position].
    Only the type's fixed slots can be constrained (variadic inputs are gathered, A-9); a fixed slot
    is constrained iff every member has a node input there and they are all distinct."""
    ops = []
    for t, members in sched:
        R = sorted(members)
        out = [R]
        nslots = fixed_slots[t]
        for j in range(nslots):
            ent = [m.inputs[v][j] for v in R]
            if any(k != "n" for k, _ in ent):
                continue
            srcs = [u for _, u in ent]
            if len(set(srcs)) != len(srcs):
                continue
            out.append(srcs)
        ops.append(out)
    return ops


def _qlike(n: PQNode) -> bool:
    return n.kind == "Q" or (n.kind == "P" and len(n.children) == 2)


def subtree_constraints(T: PQTree, O: List[int]) -> List[Tuple[int, ...]]:
    """Alg. 3 getSubtreeCons restricted to operand O, as sorted position tuples (sizes 2..|O|-1)."""
    pos = {v: i for i, v in enumerate(O)}
    node, run = T.min_subtree(O)
    out = []

    def emit(leafs):
        if 2 <= len(leafs) < len(O):
            out.append(tuple(sorted(pos[v] for v in leafs)))

    def walk(n):
        if n.kind == "L":
            return
        if n.kind == "P":
            emit(n.leafset())
        else:
            for a, b in zip(n.children, n.children[1:]):
                emit(a.leafset() | b.leafset())
        for c in n.children:
            walk(c)

    if node.kind == "Q" and run is not None:
        ch = node.children[run[0]:run[1] + 1]
        for a, b in zip(ch, ch[1:]):
            emit(a.leafset() | b.leafset())
        for c in ch:
            walk(c)
    else:
        walk(node)
    return out


def plan_pq_layout(m: Merged, sched, fixed_slots: Sequence[int], trace: Dict = None) -> Tuple[List[int], List[bool]]:
    """Returns (row_of_node, kept per batch): kept = the batch passed adjacency, broadcast and
    alignment (its constrained operands are contiguous and aligned); fixed_slots[t] = fixed input
    slots of type t.  trace (optional dict) receives "pass1" = kept per batch after the
    transactional source-constraint pass (test hook; no effect on the result)."""
    ops = batch_operands(m, sched, fixed_slots)
    T = PQTree(range(m.n))
    if m.n == 0:
        return [], []
    for o in ops:                               # results first: disjoint, always feasible
        T.reduce(o[0])
    alive = [True] * len(ops)
    for b, o in enumerate(ops):                 # sources, transactionally in schedule order
        if len(o) < 2:
            continue
        saved = copy.deepcopy(T.root)
        try:
            for S in o[1:]:
                T.reduce(S)
        except Fail:
            T.root = saved
            alive[b] = False
    if trace is not None:
        trace["pass1"] = list(alive)
    for _ in range(MAX_SWEEPS):                 # BroadcastConstraint
        any_change = False
        for b, o in enumerate(ops):
            if not alive[b] or len(o) < 2 or len(o[0]) < 2:
                continue
            cons = set()
            for O in o:
                cons.update(subtree_constraints(T, O))
            before = T.root.signature()
            saved = copy.deepcopy(T.root)
            try:
                for ps in sorted(cons):
                    for O in o:
                        T.reduce([O[i] for i in ps])
            except Fail:
                T.root = saved
                alive[b] = False
                any_change = True
                continue
            if T.root.signature() != before:
                any_change = True
        if not any_change:
            break
    return _decide_and_order(T, ops, alive, m.n), alive


def _decide_and_order(T: PQTree, ops, alive, n: int) -> List[int]:
    # canonical form (A-11)
    minleaf: Dict[int, int] = {}

    def canon(x):
        if x.kind == "L":
            minleaf[id(x)] = x.leaf
            return x.leaf
        mins = [canon(c) for c in x.children]
        if x.kind == "P":
            x.children = [c for _, c in sorted(zip(mins, x.children), key=lambda t: t[0])]
        elif mins[0] > mins[-1]:
            x.children = x.children[::-1]
        minleaf[id(x)] = min(mins)
        return minleaf[id(x)]

    canon(T.root)
    parent_of: Dict[int, PQNode] = {}
    leaf_node: Dict[int, PQNode] = {}

    def index(x):
        if x.kind == "L":
            leaf_node[x.leaf] = x
        for c in x.children:
            parent_of[id(c)] = x
            index(c)

    index(T.root)

    # extended union-find over (node, order): order(u) = tau o order(parent[u])
    uf_parent: Dict[int, int] = {}
    uf_tau: Dict[int, tuple] = {}

    def comp(a, b):  # a o b
        if len(a) == 1:
            return (a[0] * b[0],)
        return tuple(a[i] for i in b)

    def inv(a):
        if len(a) == 1:
            return a
        r = [0] * len(a)
        for i, x in enumerate(a):
            r[x] = i
        return tuple(r)

    def ident(node):
        return (1,) if _qlike(node) else tuple(range(len(node.children)))

    def find(node):
        t = ident(node)
        u = id(node)
        while u in uf_parent:
            t = comp(t, uf_tau[u])
            u = uf_parent[u]
        return u, t

    def unite(u, u2, sigma, log):
        """Alg. 5 Union for the relation order(u2) = sigma o order(u) (u, u2 nodes)."""
        r1, t1 = find(u)
        r2, t2 = find(u2)
        if r1 != r2:
            log.append(r2)
            uf_parent[r2] = r1
            uf_tau[r2] = comp(inv(t2), comp(sigma, t1))
            return True
        return t2 == comp(sigma, t1)

    def child_towards(anc, leaf):
        x = leaf_node[leaf]
        while parent_of[id(x)] is not anc:
            x = parent_of[id(x)]
        return next(i for i, c in enumerate(anc.children) if c is x)

    for b, o in enumerate(ops):
        if not alive[b] or len(o) < 2 or len(o[0]) < 2:
            continue
        log: List[int] = []
        R = o[0]
        ok = True
        r0, run0 = T.min_subtree(R)
        for O in o[1:]:
            img = dict(zip(R, O))
            r1, run1 = T.min_subtree(O)

            def match(u, u2, ru, ru2):
                if u.kind == "L" or u2.kind == "L":
                    return u.kind == "L" and u2.kind == "L" and img[u.leaf] == u2.leaf
                fu, lu = ru if ru else (0, len(u.children) - 1)
                fu2, lu2 = ru2 if ru2 else (0, len(u2.children) - 1)
                if _qlike(u) != _qlike(u2) or lu - fu != lu2 - fu2:
                    return False
                k = lu - fu + 1
                phi = []
                for t in range(k):
                    c = u.children[fu + t]
                    i2 = child_towards(u2, img[minleaf[id(c)]])
                    if not fu2 <= i2 <= lu2:
                        return False
                    phi.append(i2 - fu2)
                if _qlike(u):
                    if phi == list(range(k)):
                        sigma = (1,)
                    elif phi == list(range(k - 1, -1, -1)):
                        sigma = (-1,)
                    else:
                        return False
                else:
                    sigma = tuple(phi)
                if not unite(u, u2, sigma, log):
                    return False
                return all(match(u.children[fu + t], u2.children[fu2 + phi[t]], None, None) for t in range(k))

            if not match(r0, r1, run0, run1):
                ok = False
                break
        if not ok:
            for r2 in reversed(log):
                del uf_parent[r2]
                del uf_tau[r2]
            alive[b] = False  # alignment incompatible: this batch's sources stay gathered

    # class orientation: member with the smallest min leaf id gets identity / forward
    best: Dict[int, Tuple[int, tuple]] = {}

    def collect(x):
        if x.kind == "L":
            return
        r, t = find(x)
        if r not in best or minleaf[id(x)] < best[r][0]:
            best[r] = (minleaf[id(x)], t)
        for c in x.children:
            collect(c)

    collect(T.root)
    order: List[int] = []

    def emit(x):
        if x.kind == "L":
            order.append(x.leaf)
            return
        r, t = find(x)
        o = comp(t, inv(best[r][1]))
        if _qlike(x):
            seq = x.children if o[0] == 1 else x.children[::-1]
        else:
            seq = [x.children[i] for i in o]
        for c in seq:
            emit(c)

    emit(T.root)
    row = [0] * n
    for i, v in enumerate(order):
        row[v] = i
    return row
