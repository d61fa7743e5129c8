// ed_rl.cpp — learning the FSM batching policy by tabular N-step Q-learning (PAPER §2.3,
// P:116-140; early stop at the App. B.3 lower bound checked every 50 trials).
//
// Environment: one instance graph per episode; state S_t = E(G_t) over the ready ("frontier",
// P:123) node types; action a_t = the next batch's type; Alg. 1 then executes ALL
// ready type-a nodes.  Reward Eq. 1: r = -1 + alpha * |Frontier_a(G_t)| /
// |Frontier(G^a_t)| (A-1), where G^a is the typed subgraph of the type-a nodes whose
// edges are paths through non-a nodes (A-21) and its frontier is the unexecuted type-a nodes with
// no unexecuted G^a predecessor.  Both frontier counts are maintained incrementally.
// Update order, exploration and defaults: include/ed_batch.h and DESIGN.md A-26.
#include "ed_rl.h"

#include <algorithm>
#include <cmath>

namespace ed {
namespace {

struct SplitMix64 {
  uint64_t s;
  uint64_t next() {
    s += 0x9E3779B97F4A7C15ull;
    uint64_t z = s;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
};

// Per-instance static structure: consumers and the typed-subgraph (G^a) successors.
struct Prepared {
  std::vector<int32_t> cons_off, cons;    // consumers (CSR)
  std::vector<int32_t> gs_off, gs;        // G^{type(u)} successors of u (CSR, distinct)
  std::vector<int32_t> gpred0;            // G^{type(v)} predecessor count of v
  std::vector<int32_t> ninputs;           // node-input count
  int32_t lower_bound = 0;                // App. B.3: sum_t Depth(G^t)
};

Prepared prepare(const RlGraph &g, int nt) {
  Prepared P;
  const int n = g.n;
  P.cons_off.assign(n + 1, 0);
  P.ninputs.assign(n, 0);
  for (int v = 0; v < n; ++v) {
    P.ninputs[v] = g.pred_off[v + 1] - g.pred_off[v];
    for (int k = g.pred_off[v]; k < g.pred_off[v + 1]; ++k) ++P.cons_off[g.preds[k] + 1];
  }
  for (int v = 0; v < n; ++v) P.cons_off[v + 1] += P.cons_off[v];
  P.cons.resize(P.cons_off[n]);
  {
    std::vector<int32_t> fill(P.cons_off.begin(), P.cons_off.end() - 1);
    for (int v = 0; v < n; ++v)
      for (int k = g.pred_off[v]; k < g.pred_off[v + 1]; ++k) P.cons[fill[g.preds[k]]++] = v;
  }
  // G^a successors of u (a = type(u)): type-a nodes reached from u through non-a nodes only
  P.gs_off.assign(n + 1, 0);
  P.gpred0.assign(n, 0);
  std::vector<int32_t> mark(n, -1), stack;
  std::vector<std::vector<int32_t>> succ(n);
  for (int u = 0; u < n; ++u) {
    const int a = g.type[u];
    stack.clear();
    for (int k = P.cons_off[u]; k < P.cons_off[u + 1]; ++k) stack.push_back(P.cons[k]);
    while (!stack.empty()) {
      const int w = stack.back();
      stack.pop_back();
      if (mark[w] == u) continue;
      mark[w] = u;
      if (g.type[w] == a) {
        succ[u].push_back(w);
        ++P.gpred0[w];
      } else {
        for (int k = P.cons_off[w]; k < P.cons_off[w + 1]; ++k) stack.push_back(P.cons[k]);
      }
    }
  }
  for (int u = 0; u < n; ++u) P.gs_off[u + 1] = P.gs_off[u] + static_cast<int32_t>(succ[u].size());
  P.gs.reserve(P.gs_off[n]);
  for (int u = 0; u < n; ++u) P.gs.insert(P.gs.end(), succ[u].begin(), succ[u].end());
  // lower bound: per type, the most type-t nodes on one path (topological DP)
  std::vector<int32_t> order, rem(P.ninputs);
  for (int v = 0; v < n; ++v)
    if (rem[v] == 0) order.push_back(v);
  for (size_t q = 0; q < order.size(); ++q)
    for (int k = P.cons_off[order[q]]; k < P.cons_off[order[q] + 1]; ++k)
      if (--rem[P.cons[k]] == 0) order.push_back(P.cons[k]);
  std::vector<int32_t> cnt(n);
  for (int t = 0; t < nt; ++t) {
    int32_t best = 0;
    for (int v : order) {
      int32_t c = 0;
      for (int k = g.pred_off[v]; k < g.pred_off[v + 1]; ++k) c = std::max(c, cnt[g.preds[k]]);
      cnt[v] = c + (g.type[v] == t ? 1 : 0);
      best = std::max(best, cnt[v]);
    }
    P.lower_bound += best;
  }
  return P;
}

// Execution state of Alg. 1 on one instance.
struct Env {
  const RlGraph *g;
  const Prepared *P;
  std::vector<int32_t> remaining, grem;
  std::vector<std::vector<int32_t>> ready;  // ready nodes per type
  std::vector<int32_t> gfront;              // |Frontier(G^a_t)| per type
  int64_t left = 0;

  void reset(const RlGraph &gg, const Prepared &PP, int nt) {
    g = &gg;
    P = &PP;
    remaining = PP.ninputs;
    grem = PP.gpred0;
    ready.assign(nt, {});
    gfront.assign(nt, 0);
    for (int v = 0; v < gg.n; ++v) {
      if (remaining[v] == 0) ready[gg.type[v]].push_back(v);
      if (grem[v] == 0) ++gfront[gg.type[v]];
    }
    left = gg.n;
  }
  // frontier types -> encoded key (E_sort: descending count, ties ascending id; E_base: ascending)
  void key(int encoder, std::vector<int32_t> *k) const {
    k->clear();
    int best = -1;
    for (int t = 0; t < static_cast<int>(ready.size()); ++t)
      if (!ready[t].empty()) {
        k->push_back(t);
        if (best < 0 || ready[t].size() > ready[best].size()) best = t;  // ties: lowest id
      }
    if (encoder == ED_ENC_SORT)
      std::stable_sort(k->begin(), k->end(), [&](int a, int b) { return ready[a].size() > ready[b].size(); });
    else if (encoder == ED_ENC_MAX)
      k->push_back(best);  // E_max = (E_base, argmax type): the set, then that type
  }
  double ratio(int a) const { return static_cast<double>(ready[a].size()) / static_cast<double>(gfront[a]); }
  void execute(int a) {
    std::vector<int32_t> batch;
    batch.swap(ready[a]);
    for (int v : batch) {
      --left;
      --gfront[a];  // v leaves the frontier of G^a (a ready node has no unexecuted G^a predecessor)
      for (int k = P->gs_off[v]; k < P->gs_off[v + 1]; ++k)
        if (--grem[P->gs[k]] == 0) ++gfront[a];
      for (int k = P->cons_off[v]; k < P->cons_off[v + 1]; ++k) {
        const int w = P->cons[k];
        if (--remaining[w] == 0) ready[g->type[w]].push_back(w);
      }
    }
  }
};

int greedy(const std::map<std::pair<std::vector<int32_t>, int32_t>, double> &q, const std::vector<int32_t> &key,
           const std::vector<int32_t> &ready_types) {
  int best = -1;
  double bv = 0.0;
  for (int a : ready_types) {
    auto it = q.find({key, a});
    const double v = it == q.end() ? 0.0 : it->second;
    if (best < 0 || v > bv) { best = a; bv = v; }
  }
  return best;
}

thread_local int g_encoder = ED_ENC_SORT;  // set by rl_train: an E_max key carries its argmax type last
std::vector<int32_t> ascending(const std::vector<int32_t> &key) {
  std::vector<int32_t> r(key.begin(), key.end() - (g_encoder == ED_ENC_MAX ? 1 : 0));  // the ready types
  std::sort(r.begin(), r.end());
  return r;
}

// pi(S) = argmax_a Q(S, a) over the actions tried in S ("greedy argmax over
// ready types with table entries"); ties to the lowest type id.  Unseen pairs are valued 0 only
// while exploring (greedy() above), never in the exported table.
std::map<std::vector<int32_t>, int32_t> make_table(const std::map<std::pair<std::vector<int32_t>, int32_t>, double> &q) {
  std::map<std::vector<int32_t>, int32_t> t;
  for (const auto &kv : q) {
    auto it = t.find(kv.first.first);
    if (it == t.end()) t.emplace(kv.first.first, kv.first.second);  // actions visited ascending
    else if (kv.second > q.at({kv.first.first, it->second})) it->second = kv.first.second;
  }
  return t;
}

// Greedy Alg. 1 with the table; unseen state (or action not ready): the E_sort first type (A-3).
int64_t evaluate(const std::vector<RlGraph> &gs, const std::vector<Prepared> &Ps, int nt, int encoder,
                 const std::map<std::vector<int32_t>, int32_t> &table) {
  int64_t total = 0;
  Env env;
  std::vector<int32_t> key, skey;
  for (size_t i = 0; i < gs.size(); ++i) {
    env.reset(gs[i], Ps[i], nt);
    while (env.left > 0) {
      env.key(encoder, &key);
      env.key(ED_ENC_SORT, &skey);
      auto it = table.find(key);
      int a = it == table.end() ? -1 : it->second;
      if (a < 0 || env.ready[a].empty()) a = skey[0];
      env.execute(a);
      ++total;
    }
  }
  return total;
}

}  // namespace

std::vector<int32_t> sc_type_sequence(const RlGraph &g, int nt) {
  const Prepared P = prepare(g, nt);
  Env env;
  env.reset(g, P, nt);
  std::vector<int32_t> seq;
  while (env.left > 0) {
    int best = -1;
    double br = 0.0;
    for (int t = 0; t < nt; ++t) {
      if (env.ready[t].empty()) continue;
      const double r = env.ratio(t);
      if (best < 0 || r > br || (r == br && env.ready[t].size() > env.ready[best].size())) {
        best = t;
        br = r;
      }
    }
    seq.push_back(best);
    env.execute(best);
  }
  return seq;
}

int rl_train(const std::vector<RlGraph> &gs, int nt, const ed_rl_config_t &cfg, RlResult *out) {
  if (gs.empty() || cfg.n_steps < 1 || cfg.max_episodes < 0 || cfg.check_every < 1 || cfg.eps_every < 1 ||
      !(cfg.alpha >= 0.0) || !(cfg.lr > 0.0 && cfg.lr <= 1.0) || (cfg.encoder != ED_ENC_SORT && cfg.encoder != ED_ENC_BASE && cfg.encoder != ED_ENC_MAX) ||
      (cfg.episode_graph != ED_RL_EPISODE_INSTANCE && cfg.episode_graph != ED_RL_EPISODE_MERGED))
    return -1;
  g_encoder = cfg.encoder;
  std::vector<Prepared> Ps;
  Ps.reserve(gs.size());
  out->lower_bound = 0;
  for (const auto &g : gs) {
    Ps.push_back(prepare(g, nt));
    out->lower_bound += Ps.back().lower_bound;
  }
  SplitMix64 rng{cfg.seed};
  auto &q = out->q;
  q.clear();
  out->checkpoints.clear();
  Env env;
  struct Step { std::vector<int32_t> key; int32_t a; double r; };
  std::vector<Step> trace;
  std::vector<int32_t> key, rt;
  out->episodes = 0;
  int64_t best = -1;
  for (int ep = 0; ep < cfg.max_episodes; ++ep) {
    const size_t gi = static_cast<size_t>(ep) % gs.size();
    const double eps = std::max(cfg.eps_floor, cfg.eps0 * std::pow(cfg.eps_decay, static_cast<double>(ep / cfg.eps_every)));
    env.reset(gs[gi], Ps[gi], nt);
    trace.clear();
    while (env.left > 0) {
      env.key(cfg.encoder, &key);
      rt = ascending(key);
      const double u = static_cast<double>(rng.next() >> 11) * 0x1.0p-53;
      int a;
      if (u < eps) a = rt[rng.next() % rt.size()];
      else a = greedy(q, key, rt);
      const double r = -1.0 + cfg.alpha * env.ratio(a);
      env.execute(a);
      trace.push_back({key, a, r});
    }
    // N-step backup, t ascending (no discount)
    const int T = static_cast<int>(trace.size()), n = cfg.n_steps;
    for (int t = 0; t < T; ++t) {
      double G = 0.0;
      for (int i = 0; i < n; ++i)
        if (t + i < T) G += trace[t + i].r;
      if (t + n < T) {
        const std::vector<int32_t> &k2 = trace[t + n].key;
        double best = 0.0;
        bool first = true;
        for (int b : ascending(k2)) {
          auto it = q.find({k2, b});
          const double v = it == q.end() ? 0.0 : it->second;
          if (first || v > best) { best = v; first = false; }
        }
        G += best;
      }
      double &slot = q[{trace[t].key, trace[t].a}];  // value-initialised to 0.0 on first use
      const double old = slot;
      slot = old + cfg.lr * (G - old);
    }
    out->episodes = ep + 1;
    if ((ep + 1) % cfg.check_every == 0) {
      auto table = make_table(q);
      const int64_t total = evaluate(gs, Ps, nt, cfg.encoder, table);
      out->checkpoints.emplace_back(ep + 1, total);
      if (best < 0 || total < best) { best = total; out->table = std::move(table); }
      if (total == out->lower_bound) break;
    }
  }
  // The returned policy is the best greedy table evaluated (checkpoints, then the final Q);
  // ties keep the earlier one.  With an early stop it is the table that reached the bound.
  auto table = make_table(q);
  const int64_t total = evaluate(gs, Ps, nt, cfg.encoder, table);
  if (best < 0 || total < best) { best = total; out->table = std::move(table); }
  out->final_batches = best;
  return 0;
}

}  // namespace ed
