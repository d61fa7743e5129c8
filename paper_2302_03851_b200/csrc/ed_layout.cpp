// ed_layout.cpp — PQ-tree memory layout planner over node-output rows (host C++).
//
// PAPER.md §3.2 and App. C: a PQ tree (Booth–Lueker) holds every
// variable order in which each accepted operand is consecutive ("adjacency"); a broadcast
// pass makes the operand subtrees of each batch isomorphic (Alg. 2 BroadcastConstraint, Alg. 3);
// equivalent (node, order) pairs are unified in extended union-find sets (Alg. 4, Alg. 5); the
// leaf order is a DFS over the resolved orders (Alg. 6).  Readings (SURVEY A-9..A-13):
//   * variables = nodes; the result operand of every batch is reduced first (always feasible,
//     so every result block is contiguous); then the source operands of each batch, transactionally
//     and in schedule order (all of a batch's constraints succeed or none is kept);
//   * a source slot is constrained only if every member has a distinct node input in that slot;
//   * broadcast: round-robin sweeps over the surviving batches until a sweep changes nothing;
//     subtree constraints restricted to the operand, sets of size < 2 or == |operand| dropped;
//   * canonical form: P children sorted by min leaf id, Q oriented first-child min < last-child min;
//     union-find per batch transactionally; each class oriented so that its member with the
//     smallest min leaf id has identity / forward order.
#include "ed_layout.h"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <functional>
#include <numeric>
#include <unordered_map>
#include <vector>

namespace ed {
namespace {

enum Kind : uint8_t { LEAF = 0, PN = 1, QN = 2, DEAD = 3 };

struct Node {
  Kind kind = LEAF;
  int parent = -1;
  int leaf = -1;            // variable id (LEAF)
  int nleaves = 1;
  std::vector<int> ch;      // children (P: unordered, Q: ordered)
};

class PQTree {
 public:
  explicit PQTree(int n) {
    nodes_.resize(n + 1);
    for (int v = 0; v < n; ++v) {
      nodes_[v].kind = LEAF;
      nodes_[v].leaf = v;
      nodes_[v].parent = n;
      nodes_[v].nleaves = 1;
    }
    Node &r = nodes_[n];
    r.kind = n >= 2 ? PN : (n == 1 ? LEAF : PN);
    if (n >= 2) {
      r.ch.resize(n);
      std::iota(r.ch.begin(), r.ch.end(), 0);
      r.nleaves = n;
      root_ = n;
    } else if (n == 1) {
      nodes_.pop_back();
      nodes_[0].parent = -1;
      root_ = 0;
    } else {
      root_ = -1;
    }
    cnt_.assign(nodes_.size(), 0);
  }

  int root() const { return root_; }
  const Node &node(int id) const { return nodes_[id]; }
  int size() const { return static_cast<int>(nodes_.size()); }

  // ---- transactions (undo log) ----
  void begin() {
    in_txn_ = true;
    saved_size_ = nodes_.size();
    saved_root_ = root_;
    log_.clear();
    logged_.clear();
  }
  // A committed transaction that changed the tree stamps every node it modified or created with a
  // new epoch: a batch whose operand subtrees carry no stamp newer than its last processing cannot
  // derive new broadcast constraints (A-10: such a batch may be skipped, results are identical).
  void commit() {
    if (changed_since_begin()) {
      ++epoch_;
      stamp_.resize(nodes_.size(), 0);
      for (const auto &e : log_) stamp_[e.first] = epoch_;
      for (size_t id = saved_size_; id < nodes_.size(); ++id) stamp_[id] = epoch_;
    }
    in_txn_ = false;
    log_.clear();
    logged_.clear();
  }
  uint32_t epoch() const { return epoch_; }
  // newest stamp in the subtree of r (children f..l only when r is a partial Q run)
  uint32_t subtree_stamp(int r, int f, int l) const {
    uint32_t m = stamp_of(r);
    std::vector<int> st;
    const auto &ch = nodes_[r].ch;
    if (nodes_[r].kind == QN) {
      for (int k = f; k <= l; ++k) st.push_back(ch[k]);
    } else {
      st.assign(ch.begin(), ch.end());
    }
    while (!st.empty()) {
      const int x = st.back();
      st.pop_back();
      m = std::max(m, stamp_of(x));
      for (int c : nodes_[x].ch) st.push_back(c);
    }
    return m;
  }
  void rollback() {
    for (auto it = log_.rbegin(); it != log_.rend(); ++it) nodes_[it->first] = it->second;
    nodes_.resize(saved_size_);
    root_ = saved_root_;
    in_txn_ = false;
    log_.clear();
    logged_.clear();
    cnt_.resize(nodes_.size());
  }
  bool changed_since_begin() const { return !log_.empty() || nodes_.size() != saved_size_ || root_ != saved_root_; }

  // Reduce: restrict the frontier to orders where the leaves of S are consecutive.  Returns false
  // if impossible (the tree is then in an undefined state: the caller rolls the transaction back).
  bool reduce(const std::vector<int> &S) {
    if (S.size() <= 1) return true;
    // pertinent counts along root paths
    touched_.clear();
    for (int v : S) {
      for (int x = v; x != -1; x = nodes_[x].parent) {
        if (cnt_[x] == 0) touched_.push_back(x);
        ++cnt_[x];
      }
    }
    const int s = static_cast<int>(S.size());
    int proot = S[0];
    while (cnt_[proot] < s) proot = nodes_[proot].parent;
    bool ok = process(proot, true, s);
    for (int x : touched_) if (x < static_cast<int>(cnt_.size())) cnt_[x] = 0;
    for (int x : extra_cnt_) if (x < static_cast<int>(cnt_.size())) cnt_[x] = 0;
    extra_cnt_.clear();
    if (ok) normalize();
    return ok;
  }

  // leaves of the subtree of id, in current order
  void leaves(int id, std::vector<int> &out) const {
    if (nodes_[id].kind == LEAF) { out.push_back(nodes_[id].leaf); return; }
    for (int c : nodes_[id].ch) leaves(c, out);
  }

  // Minimal subtree holding exactly the (consecutive) leaf set S: (root, first, last) where
  // [first, last] is the covered run of root's children (whole node: 0 .. size-1).
  void min_subtree(const std::vector<int> &S, int *r, int *first, int *last) {
    touched_.clear();
    for (int v : S)
      for (int x = v; x != -1; x = nodes_[x].parent) {
        if (cnt_[x] == 0) touched_.push_back(x);
        ++cnt_[x];
      }
    const int s = static_cast<int>(S.size());
    int x = S[0];
    while (cnt_[x] < s) x = nodes_[x].parent;
    *r = x;
    *first = -1;
    *last = -1;
    if (nodes_[x].kind != LEAF) {
      const auto &ch = nodes_[x].ch;
      for (int k = 0; k < static_cast<int>(ch.size()); ++k)
        if (cnt_[ch[k]] > 0) {
          if (*first < 0) *first = k;
          *last = k;
        }
    }
    for (int t : touched_) cnt_[t] = 0;
  }

  int child_index_towards(int anc, int leafnode) const {
    int x = leafnode;
    while (nodes_[x].parent != anc) {
      x = nodes_[x].parent;
      if (x < 0) return -1;
    }
    const auto &ch = nodes_[anc].ch;
    for (int k = 0; k < static_cast<int>(ch.size()); ++k)
      if (ch[k] == x) return k;
    return -1;
  }

  void set_children(int id, std::vector<int> ch) { nodes_[id].ch = std::move(ch); }

  // debug: structural invariants (parent links, leaf counts, no dead node reachable, arity)
  const char *check() const {
    if (root_ < 0) return nullptr;
    if (nodes_[root_].parent != -1) return "root has a parent";
    std::vector<int> st = {root_};
    int leaves = 0;
    while (!st.empty()) {
      const int x = st.back();
      st.pop_back();
      const Node &n = nodes_[x];
      if (n.kind == DEAD) return "dead node reachable";
      if (n.kind == LEAF) { ++leaves; if (n.nleaves != 1) return "leaf nleaves"; continue; }
      if (n.ch.size() < 2) return "internal node with < 2 children";
      int sum = 0;
      for (int c : n.ch) {
        if (nodes_[c].parent != x) return "bad parent link";
        sum += nodes_[c].nleaves;
        st.push_back(c);
      }
      if (sum != n.nleaves) return "nleaves mismatch";
    }
    return nullptr;
  }

 private:
  std::vector<Node> nodes_;
  int root_ = -1;
  std::vector<int> cnt_, touched_, extra_cnt_;
  bool in_txn_ = false;
  size_t saved_size_ = 0;
  int saved_root_ = -1;
  std::vector<std::pair<int, Node>> log_;
  std::vector<char> logged_;
  std::vector<uint32_t> stamp_;
  uint32_t epoch_ = 0;
  uint32_t stamp_of(int id) const { return id < static_cast<int>(stamp_.size()) ? stamp_[id] : 0; }

  void touch(int id) {
    if (!in_txn_ || id >= static_cast<int>(saved_size_)) return;
    if (static_cast<int>(logged_.size()) <= id) logged_.resize(nodes_.size(), 0);
    if (logged_[id]) return;
    logged_[id] = 1;
    log_.emplace_back(id, nodes_[id]);
  }
  int new_node(Kind k, std::vector<int> ch) {
    Node n;
    n.kind = k;
    n.nleaves = 0;
    for (int c : ch) n.nleaves += nodes_[c].nleaves;
    n.ch = std::move(ch);
    nodes_.push_back(std::move(n));
    const int id = static_cast<int>(nodes_.size()) - 1;
    cnt_.push_back(0);
    for (int c : nodes_[id].ch) {
      touch(c);
      nodes_[c].parent = id;
    }
    modified_.push_back(id);
    return id;
  }
  // one node for a group of children (the child itself if there is one)
  int group(Kind k, const std::vector<int> &g) { return g.size() == 1 ? g[0] : new_node(k, g); }

  void replace_child(int parent, int oldc, int newc) {
    if (parent < 0) {
      root_ = newc;
      touch(newc);
      nodes_[newc].parent = -1;
      return;
    }
    touch(parent);
    for (int &c : nodes_[parent].ch)
      if (c == oldc) c = newc;
    touch(newc);
    nodes_[newc].parent = parent;
    modified_.push_back(parent);
  }
  void set_kids(int id, std::vector<int> ch) {
    if (ch == nodes_[id].ch) return;  // no structural change
    touch(id);
    nodes_[id].ch = std::move(ch);
    int nl = 0;
    for (int c : nodes_[id].ch) {
      touch(c);
      nodes_[c].parent = id;
      nl += nodes_[c].nleaves;
    }
    nodes_[id].nleaves = nl;
    modified_.push_back(id);
  }
  void kill(int id) {
    touch(id);
    nodes_[id].kind = DEAD;
    nodes_[id].ch.clear();
  }

  std::vector<int> modified_;
  // label after processing: 0 empty, 1 full, 2 partial (Q with [empty..., full...])

  // Post-order template application on the pertinent subtree.  Non-root nodes return their label
  // (a partial node becomes a Q-node ordered empty -> full); the root applies the root templates.
  // Returns false on failure.
  bool process(int x, bool is_root, int s) {
    if (cnt_[x] == nodes_[x].nleaves) return true;  // full (or the pertinent root is full: nothing to do)
    Node &X = nodes_[x];
    if (X.kind == LEAF) return true;
    // recurse into partial children first (full / empty children need no work)
    std::vector<int> kids = X.ch;
    for (int c : kids)
      if (cnt_[c] > 0 && cnt_[c] < nodes_[c].nleaves)
        if (!process(c, false, s)) return false;
    // children may have been replaced: re-read
    kids = nodes_[x].ch;
    std::vector<int> E, F, Pt;
    std::vector<int> lab(kids.size());
    for (size_t k = 0; k < kids.size(); ++k) {
      const int c = kids[k];
      lab[k] = cnt_[c] == 0 ? 0 : (cnt_[c] == nodes_[c].nleaves ? 1 : 2);
      (lab[k] == 0 ? E : (lab[k] == 1 ? F : Pt)).push_back(c);
    }
    const int parent = nodes_[x].parent;
    if (nodes_[x].kind == PN) {
      if (!is_root) {
        if (Pt.empty()) {  // P3: Q [P(E), P(F)]
          const int e = group(PN, E), f = group(PN, F);
          const int q = new_node(QN, {e, f});
          cnt_[q] = cnt_[x];
          extra_cnt_.push_back(q);
          replace_child(parent, x, q);
          kill(x);
          return true;
        }
        if (Pt.size() == 1) {  // P5: Q [P(E), Y..., P(F)]
          const int y = Pt[0];
          std::vector<int> seq;
          if (!E.empty()) seq.push_back(group(PN, E));
          for (int c : nodes_[y].ch) seq.push_back(c);
          if (!F.empty()) seq.push_back(group(PN, F));
          const int q = new_node(QN, seq);
          cnt_[q] = cnt_[x];
          extra_cnt_.push_back(q);
          replace_child(parent, x, q);
          kill(x);
          kill(y);
          return true;
        }
        return false;
      }
      // pertinent root P-node
      if (Pt.empty()) {  // P2
        if (F.size() >= 2 && !E.empty()) {
          const int f = new_node(PN, F);
          cnt_[f] = 0;
          std::vector<int> nk = E;
          nk.push_back(f);
          set_kids(x, nk);
        }
        return true;
      }
      if (Pt.size() == 1) {  // P4
        const int y = Pt[0];
        std::vector<int> ych = nodes_[y].ch;
        if (!F.empty()) ych.push_back(group(PN, F));
        set_kids(y, ych);
        if (E.empty()) {
          replace_child(parent, x, y);
          kill(x);
        } else {
          std::vector<int> nk = E;
          nk.push_back(y);
          set_kids(x, nk);
        }
        return true;
      }
      if (Pt.size() == 2) {  // P6
        const int y1 = Pt[0], y2 = Pt[1];
        std::vector<int> seq = nodes_[y1].ch;
        if (!F.empty()) seq.push_back(group(PN, F));
        const std::vector<int> &c2 = nodes_[y2].ch;
        for (auto it = c2.rbegin(); it != c2.rend(); ++it) seq.push_back(*it);
        const int q = new_node(QN, seq);
        kill(y1);
        kill(y2);
        if (E.empty()) {
          replace_child(parent, x, q);
          kill(x);
        } else {
          std::vector<int> nk = E;
          nk.push_back(q);
          set_kids(x, nk);
        }
        return true;
      }
      return false;
    }
    // Q-node
    const int k = static_cast<int>(kids.size());
    if (!is_root) {
      // need [E*, P?, F*] with the pertinent part at one end (possibly after reversal)
      auto try_dir = [&](bool rev) -> bool {
        std::vector<int> ord(k);
        for (int i = 0; i < k; ++i) ord[i] = rev ? k - 1 - i : i;
        int i = 0;
        while (i < k && lab[ord[i]] == 0) ++i;
        int npart = 0;
        if (i < k && lab[ord[i]] == 2) { ++npart; ++i; }
        while (i < k && lab[ord[i]] == 1) ++i;
        if (i != k) return false;
        std::vector<int> seq;
        for (int t = 0; t < k; ++t) {
          const int c = kids[ord[t]];
          if (lab[ord[t]] == 2) for (int cc : nodes_[c].ch) seq.push_back(cc);
          else seq.push_back(c);
        }
        for (int t = 0; t < k; ++t) if (lab[ord[t]] == 2) kill(kids[ord[t]]);
        set_kids(x, seq);
        return true;
      };
      return try_dir(false) || try_dir(true);
    }
    // pertinent root Q-node: [E*, P?, F*, P?, E*]
    int a = 0;
    while (a < k && lab[a] == 0) ++a;
    int b = k - 1;
    while (b >= 0 && lab[b] == 0) --b;
    for (int t = a; t <= b; ++t) {
      if (lab[t] == 0) return false;
      if (lab[t] == 2 && t != a && t != b) return false;
    }
    std::vector<int> seq;
    for (int t = 0; t < k; ++t) {
      const int c = kids[t];
      if (lab[t] == 2) {
        const auto &cc = nodes_[c].ch;
        if (t == a && a != b) for (int z : cc) seq.push_back(z);                       // empty .. full
        else if (t == b && a != b) for (auto it = cc.rbegin(); it != cc.rend(); ++it) seq.push_back(*it);
        else return false;  // a lone partial child cannot be the pertinent root's only pertinent part
      } else {
        seq.push_back(c);
      }
    }
    for (int t = a; t <= b; ++t) if (lab[t] == 2) kill(kids[t]);
    set_kids(x, seq);
    return true;
  }

  // Collapse 1-child nodes and turn 2-child Q-nodes into P-nodes (canonical Booth–Lueker form).
  void normalize() {
    std::vector<int> mods;
    mods.swap(modified_);
    for (int id : mods) {
      if (id >= static_cast<int>(nodes_.size()) || nodes_[id].kind == DEAD || nodes_[id].kind == LEAF) continue;
      Node &n = nodes_[id];
      if (n.ch.size() == 2 && n.kind == QN) {
        touch(id);
        nodes_[id].kind = PN;
      }
      // splice a P child into a P parent? (keep: a P child of a P node is a real constraint)
      if (nodes_[id].ch.size() == 1) {
        const int c = nodes_[id].ch[0];
        replace_child(nodes_[id].parent, id, c);
        kill(id);
      }
    }
    modified_.clear();
  }
};

// ------------------------------------------------------------------------------------------------
// extended union-find (Alg. 5): element = (node, order); Find(u) = (root, tau) with
// order(u) = tau o order(root).  Q: tau in {+1, -1}; P: tau a permutation of canonical child indices.
// ------------------------------------------------------------------------------------------------
struct UF {
  std::unordered_map<int, int> parent;
  std::unordered_map<int, std::vector<int>> tau;  // transform to parent (P: permutation; Q: {+1|-1})
  std::vector<std::pair<int, std::pair<int, std::vector<int>>>> log;  // undo: (node, (old parent, old tau))
  bool logging = false;

  int par(int u) const {
    auto it = parent.find(u);
    return it == parent.end() ? u : it->second;
  }
  static std::vector<int> compose(const std::vector<int> &a, const std::vector<int> &b) {  // a o b
    if (a.size() == 1) return {a[0] * b[0]};
    std::vector<int> r(b.size());
    for (size_t k = 0; k < b.size(); ++k) r[k] = a[b[k]];
    return r;
  }
  static std::vector<int> inverse(const std::vector<int> &a) {
    if (a.size() == 1) return a;
    std::vector<int> r(a.size());
    for (size_t k = 0; k < a.size(); ++k) r[a[k]] = static_cast<int>(k);
    return r;
  }
  static std::vector<int> identity(int k, bool q) {
    if (q) return {1};
    std::vector<int> r(k);
    std::iota(r.begin(), r.end(), 0);
    return r;
  }
  // (root, tau) with order(u) = tau o order(root)
  std::pair<int, std::vector<int>> find(int u, int k, bool q) const {
    std::vector<int> t = identity(k, q);
    while (true) {
      auto it = parent.find(u);
      if (it == parent.end()) return {u, t};
      t = compose(t, tau.at(u));
      u = it->second;
    }
  }
  // relation order(u2) = sigma o order(u1)
  bool unite(int u1, int u2, const std::vector<int> &sigma, int k, bool q) {
    auto [r1, t1] = find(u1, k, q);
    auto [r2, t2] = find(u2, k, q);
    if (r1 != r2) {
      // order(r2) = t2^-1 o sigma o t1 o order(r1)
      std::vector<int> T = compose(inverse(t2), compose(sigma, t1));
      if (logging) {
        auto it = parent.find(r2);
        log.push_back({r2, {it == parent.end() ? -1 : it->second, it == parent.end() ? std::vector<int>{} : tau[r2]}});
      }
      parent[r2] = r1;
      tau[r2] = T;
      return true;
    }
    return t2 == compose(sigma, t1);
  }
  void rollback() {
    for (auto it = log.rbegin(); it != log.rend(); ++it) {
      if (it->second.first < 0) {
        parent.erase(it->first);
        tau.erase(it->first);
      } else {
        parent[it->first] = it->second.first;
        tau[it->first] = it->second.second;
      }
    }
    log.clear();
  }
};

// A node whose order is a direction: a Q-node, or a 2-child P-node (its two orders are the two
// directions; Booth–Lueker keeps 2-child nodes as P-nodes, a 2-element Q run is directional too).
bool qlike(const Node &n) { return n.kind == QN || (n.kind == PN && n.ch.size() == 2); }

}  // namespace

std::vector<int32_t> plan_layout_pq(const LayoutInput &in) {
  const int V = static_cast<int>(in.V);
  const auto &gtype = *in.gtype;
  const auto &in_off = *in.in_off;
  const auto &in_idx = *in.in_idx;
  const auto &bo = *in.batch_off;
  const auto &mem = *in.members;
  const auto &types = *in.types;
  const int nb = static_cast<int>(in.batch_type->size());
  if (V == 0) return {};

  // operands per batch: ops[b][0] = result (members in ascending id), ops[b][j] = constrained slots
  std::vector<std::vector<std::vector<int>>> ops(nb);
  for (int b = 0; b < nb; ++b) {
    std::vector<int> R(mem.begin() + bo[b], mem.begin() + bo[b + 1]);
    std::sort(R.begin(), R.end());
    ops[b].push_back(R);
    const ed_op_type_t &ot = types[gtype[R[0]]];
    for (int j = 0; j < ot.num_slots; ++j) {
      std::vector<int> S(R.size());
      bool ok = true;
      for (size_t i = 0; i < R.size() && ok; ++i) {
        const int x = in_idx[in_off[R[i]] + j];
        if (x < 0) ok = false;
        S[i] = x;
      }
      if (!ok) continue;
      std::vector<int> srt = S;
      std::sort(srt.begin(), srt.end());
      if (std::adjacent_find(srt.begin(), srt.end()) != srt.end()) continue;  // repeated input: broadcast-like
      ops[b].push_back(S);
    }
  }

  const bool dbg = std::getenv("ED_PQ_DEBUG") != nullptr;
  auto now = [] { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count(); };
  double t0 = now();
  PQTree T(V);
  // results first (disjoint: always feasible)
  for (int b = 0; b < nb; ++b) {
    T.begin();
    if (!T.reduce(ops[b][0])) T.rollback(); else T.commit();
  }
  std::vector<char> alive(nb, 1);
  for (int b = 0; b < nb; ++b) {
    if (ops[b].size() < 2) continue;
    T.begin();
    bool ok = true;
    for (size_t j = 1; j < ops[b].size() && ok; ++j) ok = T.reduce(ops[b][j]);
    if (ok) T.commit(); else { T.rollback(); alive[b] = 0; }
    if (dbg) if (const char *e = T.check()) std::fprintf(stderr, "[pq] after source batch %d (%s): %s\n", b, ok ? "ok" : "rolled back", e);
  }
  double t1 = now();
  int sweeps = 0;
  double t_derive = 0, t_reduce = 0;
  // BroadcastConstraint: sweeps until no batch changes the tree.  A batch whose operand subtrees
  // are unchanged since its last processing is skipped (A-10: its constraints are already applied).
  std::vector<int64_t> done_epoch(nb, -1);
  int64_t skipped = 0;
  for (int sweep = 0; sweep < 200; ++sweep) {
    ++sweeps;
    bool any = false;
    for (int b = 0; b < nb; ++b) {
      if (!alive[b] || ops[b].size() < 2) continue;
      const int m = static_cast<int>(ops[b][0].size());
      if (m < 2) continue;
      if (done_epoch[b] >= 0) {
        uint32_t newest = 0;
        for (const auto &O : ops[b]) {
          int r, f, l;
          T.min_subtree(O, &r, &f, &l);
          newest = std::max(newest, T.subtree_stamp(r, f, l));
        }
        if (static_cast<int64_t>(newest) <= done_epoch[b]) {
          ++skipped;
          continue;
        }
      }
      const double td0 = dbg ? now() : 0;
      // position of each variable in each operand
      std::vector<std::vector<int>> cons;  // position sets
      for (size_t o = 0; o < ops[b].size(); ++o) {
        const auto &O = ops[b][o];
        std::unordered_map<int, int> pos;
        pos.reserve(O.size() * 2);
        for (int i = 0; i < m; ++i) pos[O[i]] = i;
        int r, f, l;
        T.min_subtree(O, &r, &f, &l);
        // getSubtreeCons (Alg. 3): P-node -> its leaves; Q-node -> each adjacent sibling pair
        std::vector<int> stack;
        auto emit = [&](const std::vector<int> &leafs) {
          if (leafs.size() < 2 || static_cast<int>(leafs.size()) == m) return;
          std::vector<int> ps;
          for (int v : leafs) ps.push_back(pos.at(v));
          std::sort(ps.begin(), ps.end());
          cons.push_back(ps);
        };
        std::function<void(int)> walk = [&](int id) {
          const Node &n = T.node(id);
          if (n.kind == LEAF) return;
          if (n.kind == PN) {
            std::vector<int> lv;
            T.leaves(id, lv);
            emit(lv);
          } else {
            for (size_t k = 0; k + 1 < n.ch.size(); ++k) {
              std::vector<int> lv;
              T.leaves(n.ch[k], lv);
              T.leaves(n.ch[k + 1], lv);
              emit(lv);
            }
          }
          for (int c : n.ch) walk(c);
        };
        if (T.node(r).kind == QN && !(f == 0 && l == static_cast<int>(T.node(r).ch.size()) - 1)) {
          const auto &ch = T.node(r).ch;
          for (int k = f; k < l; ++k) {
            std::vector<int> lv;
            T.leaves(ch[k], lv);
            T.leaves(ch[k + 1], lv);
            emit(lv);
          }
          for (int k = f; k <= l; ++k) walk(ch[k]);
        } else {
          walk(r);
        }
      }
      std::sort(cons.begin(), cons.end());
      cons.erase(std::unique(cons.begin(), cons.end()), cons.end());
      const double td1 = dbg ? now() : 0;
      t_derive += td1 - td0;
      T.begin();
      bool ok = true;
      for (const auto &ps : cons) {
        for (size_t o = 0; o < ops[b].size() && ok; ++o) {
          std::vector<int> S;
          for (int pidx : ps) S.push_back(ops[b][o][pidx]);
          ok = T.reduce(S);
        }
        if (!ok) break;
      }
      if (dbg) t_reduce += now() - td1;
      if (!ok) {
        T.rollback();
        alive[b] = 0;
        any = true;
      } else {
        if (T.changed_since_begin()) any = true;
        T.commit();
        done_epoch[b] = T.epoch();
      }
      if (dbg) if (const char *e = T.check()) std::fprintf(stderr, "[pq] sweep %d batch %d (%s): %s\n", sweep, b, ok ? "ok" : "rolled back", e);
    }
    if (!any) break;
  }

  double t2 = now();
  // canonical form (A-11): min leaf id per node; P children sorted by it; Q first-child min < last
  std::vector<int> minleaf(T.size(), INT32_MAX);
  std::function<int(int)> mn = [&](int id) -> int {
    const Node &n = T.node(id);
    int v = n.kind == LEAF ? n.leaf : INT32_MAX;
    for (int c : n.ch) v = std::min(v, mn(c));
    minleaf[id] = v;
    return v;
  };
  const int root = T.root();
  mn(root);
  std::function<void(int)> canon = [&](int id) {
    const Node &n = T.node(id);
    if (n.kind == LEAF) return;
    std::vector<int> ch = n.ch;
    if (n.kind == PN) {
      std::sort(ch.begin(), ch.end(), [&](int a, int c) { return minleaf[a] < minleaf[c]; });
    } else if (minleaf[ch.front()] > minleaf[ch.back()]) {
      std::reverse(ch.begin(), ch.end());
    }
    T.set_children(id, ch);
    for (int c : ch) canon(c);
  };
  canon(root);

  // DecideNodesOrder (Alg. 4 / Alg. 5), per batch transactionally
  UF uf;
  for (int b = 0; b < nb; ++b) {
    if (!alive[b] || ops[b].size() < 2 || ops[b][0].size() < 2) continue;
    uf.log.clear();
    uf.logging = true;
    bool ok = true;
    const auto &R = ops[b][0];
    int r0, f0, l0;
    T.min_subtree(R, &r0, &f0, &l0);
    for (size_t o = 1; o < ops[b].size() && ok; ++o) {
      const auto &O = ops[b][o];
      std::unordered_map<int, int> img;  // result leaf -> operand leaf (same position)
      for (size_t i = 0; i < R.size(); ++i) img[R[i]] = O[i];
      int r1, f1, l1;
      T.min_subtree(O, &r1, &f1, &l1);
      // simultaneous walk: (u in R's subtree, u' in O's subtree, covered run of u)
      std::function<bool(int, int, int, int, int, int)> match = [&](int u, int u2, int fu, int lu, int fu2,
                                                                    int lu2) -> bool {
        const Node &A = T.node(u), &B = T.node(u2);
        if (A.kind == LEAF || B.kind == LEAF) {
          return A.kind == LEAF && B.kind == LEAF && img.at(A.leaf) == B.leaf;
        }
        if (qlike(A) != qlike(B) || lu - fu != lu2 - fu2) return false;
        const int k = lu - fu + 1;
        std::vector<int> phi(k);
        for (int t = 0; t < k; ++t) {
          const int c = A.ch[fu + t];
          const int y = img.at(minleaf[c]);  // any leaf of c; its image lies in the matching child
          const int idx = T.child_index_towards(u2, y);
          if (idx < fu2 || idx > lu2) return false;
          phi[t] = idx - fu2;
        }
        const bool q = qlike(A);
        std::vector<int> sigma;
        if (q) {
          bool idn = true, rev = true;
          for (int t = 0; t < k; ++t) {
            idn &= phi[t] == t;
            rev &= phi[t] == k - 1 - t;
          }
          if (!idn && !rev) return false;
          sigma = {idn ? 1 : -1};
        } else {
          sigma = phi;
        }
        if (!uf.unite(u, u2, sigma, static_cast<int>(A.ch.size()), q)) return false;
        for (int t = 0; t < k; ++t) {
          const int c = A.ch[fu + t], c2 = B.ch[fu2 + phi[t]];
          const int nc = T.node(c).kind == LEAF ? 0 : static_cast<int>(T.node(c).ch.size()) - 1;
          const int nc2 = T.node(c2).kind == LEAF ? 0 : static_cast<int>(T.node(c2).ch.size()) - 1;
          if (!match(c, c2, 0, nc, 0, nc2)) return false;
        }
        return true;
      };
      const int nr0 = T.node(r0).kind == LEAF ? 0 : static_cast<int>(T.node(r0).ch.size()) - 1;
      const int nr1 = T.node(r1).kind == LEAF ? 0 : static_cast<int>(T.node(r1).ch.size()) - 1;
      ok = match(r0, r1, f0 < 0 ? 0 : f0, l0 < 0 ? nr0 : l0, f1 < 0 ? 0 : f1, l1 < 0 ? nr1 : l1);
    }
    if (!ok) uf.rollback();
    uf.logging = false;
    uf.log.clear();
  }

  // class orientation: the member with the smallest min leaf id gets identity / forward
  std::unordered_map<int, std::pair<int, std::vector<int>>> best;  // class root -> (min leaf, tau of member)
  std::function<void(int)> collect = [&](int id) {
    const Node &n = T.node(id);
    if (n.kind == LEAF) return;
    const bool q = qlike(n);
    auto [r, t] = uf.find(id, static_cast<int>(n.ch.size()), q);
    auto it = best.find(r);
    if (it == best.end() || minleaf[id] < it->second.first) best[r] = {minleaf[id], t};
    for (int c : n.ch) collect(c);
  };
  collect(root);
  std::vector<int32_t> order;
  order.reserve(V);
  std::function<void(int)> emit = [&](int id) {
    const Node &n = T.node(id);
    if (n.kind == LEAF) { order.push_back(n.leaf); return; }
    const bool q = qlike(n);
    const int k = static_cast<int>(n.ch.size());
    auto [r, t] = uf.find(id, k, q);
    // order(root) = tau_best^-1  =>  order(id) = t o tau_best^-1
    const std::vector<int> o = UF::compose(t, UF::inverse(best.at(r).second));
    if (q) {
      if (o[0] == 1) for (int c : n.ch) emit(c);
      else for (auto it2 = n.ch.rbegin(); it2 != n.ch.rend(); ++it2) emit(*it2);
    } else {
      for (int pos = 0; pos < k; ++pos) emit(n.ch[o[pos]]);
    }
  };
  emit(root);
  std::vector<int32_t> row(V, -1);
  for (int i = 0; i < V; ++i) row[order[i]] = i;
  if (dbg) {
    int nalive = 0;
    for (int b = 0; b < nb; ++b) nalive += alive[b] && ops[b].size() > 1;
    std::fprintf(stderr, "[pq] broadcast: derive %.1f ms, reduce %.1f ms, %lld batch visits skipped\n", t_derive,
                 t_reduce, static_cast<long long>(skipped));
    std::fprintf(stderr, "[pq] construct %.1f ms, broadcast %.1f ms (%d sweeps), order %.1f ms, alive %d/%d\n", t1 - t0,
                 t2 - t1, sweeps, now() - t2, nalive, nb);
  }
  return row;
}

}  // namespace ed
