// ed_batch.cpp — host side of libedbatch.so: C ABI (include/ed_batch.h), graph ingest and
// validation, Alg. 1 FSM frontier scheduler, layout planning, lowering to the device step table.
//
// PAPER.md references: Alg. 1; types; E_sort; policy lookup;
// lower bound (App. B.3); memory layout (§3).  Readings: DESIGN.md §3.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>
#include <algorithm>

#include <cuda_runtime.h>

#include "ed_batch.h"
#include "ed_internal.h"
#include "ed_layout.h"
#include "ed_rl.h"

namespace {

thread_local std::string g_last_error;

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void *p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// 2-D bf16 row-major [rows x cols] tensor map with 128B swizzle, box {64, box_rows}.
bool encode_rows(CUtensorMap *m, const void *base, int64_t rows, int64_t cols, uint32_t box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn || !base || rows <= 0) return false;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols) * 2};
  cuuint32_t box[2] = {64, box_rows}, es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

ed_status_t fail(ed_status_t code, const std::string &msg) {
  g_last_error = msg;
  return code;
}

double now_us() {
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Pinned staging buffers for the async H2D upload of a plan's static part (step table, index
// arrays): a ring of kStagingSlots buffers, so the host can upload the next minibatches' plans
// while earlier kernels still run on the stream (a slot is reused once the copy recorded on it has
// completed; with one buffer every upload waited for the previous kernel).  A new minibatch plan
// needs no cudaMallocHost.
constexpr int kStagingSlots = 4;
struct StagingSlot {
  void *buf = nullptr;
  size_t cap = 0;
  cudaEvent_t done = nullptr;
  bool pending = false;
};
struct Staging {
  std::mutex mu;
  StagingSlot slot[kStagingSlots];
  int next = 0;
};
Staging &staging() {
  static Staging s;
  return s;
}

cudaError_t upload_async(void *dst, const void *src, size_t n, cudaStream_t s) {
  Staging &stg = staging();
  std::lock_guard<std::mutex> lk(stg.mu);
  StagingSlot &st = stg.slot[stg.next];
  stg.next = (stg.next + 1) % kStagingSlots;
  cudaError_t e = cudaSuccess;
  if (st.pending) {
    e = cudaEventSynchronize(st.done);
    if (e != cudaSuccess) return e;
    st.pending = false;
  }
  if (n > st.cap) {
    if (st.buf) cudaFreeHost(st.buf);
    st.cap = std::max<size_t>(n, size_t(4) << 20);
    e = cudaMallocHost(&st.buf, st.cap);
    if (e != cudaSuccess) { st.buf = nullptr; st.cap = 0; return e; }
  }
  if (!st.done) {
    e = cudaEventCreateWithFlags(&st.done, cudaEventDisableTiming);
    if (e != cudaSuccess) return e;
  }
  std::memcpy(st.buf, src, n);
  e = cudaMemcpyAsync(dst, st.buf, n, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return e;
  e = cudaEventRecord(st.done, s);
  st.pending = (e == cudaSuccess);
  return e;
}

// Which plan's static part currently sits in which workspace (a workspace can be shared by
// several plans; the step table is re-uploaded whenever the owner changes).
struct WsBinding {
  const void *plan = nullptr;
  uint64_t nonce = 0;  // written into the workspace header at binding, checked by every launch
  uint32_t seq = 0;    // launches since the binding (readiness counters are monotonic)
};
struct WsRegistry {
  std::mutex mu;
  std::map<const void *, WsBinding> owner;  // workspace -> binding
  // workspace -> event recorded on the launch stream after its last launch (kept for the process:
  // an upload on a side stream waits for it before overwriting the workspace's static part)
  std::map<const void *, cudaEvent_t> done;
  cudaEvent_t up_ev[16] = {};  // ring of events ordering side-stream uploads before their launches
  int up_next = 0;
  uint64_t next_nonce = 0x5EDB000000000001ull;
};
WsRegistry &ws_registry() {
  static WsRegistry r;
  return r;
}

}  // namespace

struct ed_plan_s {
  // types
  std::vector<ed_op_type_t> types;
  int hidden = 0, dtype = 0;
  // merged graph (global ids)
  int64_t V = 0;
  int32_t ninst = 0;
  std::vector<int32_t> gtype, in_off, in_idx, ext;  // in_idx: >=0 global node, ZERO, or -1-id external
  std::vector<int32_t> indeg, coff, cons;  // node-input counts and consumers CSR (from validation)
  std::vector<int32_t> roots;                         // global node id or -1-id
  // schedule
  std::vector<int32_t> batch_type, batch_off, members;
  int64_t lower_bound = 0;
  // layout
  std::vector<int32_t> row_of_node;
  std::vector<int32_t> slot_modes;
  // lowering
  std::vector<ed::DevStep> steps;
  std::vector<int32_t> step_batch;   // schedule batch of every device step
  bool level_order = true;           // ED_ORDER_LEVEL
  std::vector<int32_t> idx;
  std::vector<int32_t> root_rows;
  std::vector<int32_t> target;  // per row: sum of ed::step_contrib over the device steps writing it
  int root_wset = 0;
  // workspace layout
  size_t off_bar = 0, off_ts = 0, off_steps = 0, off_idx = 0, off_roots = 0, off_target = 0, off_ready = 0,
         off_h = 0, off_c = 0, off_y = 0, off_x = 0, off_u = 0, off_m = 0, ws_bytes = 0;
  int64_t y_cols = 0;
  bool need_x = false;
  bool has_split = false;   // some step is split-K over a CTA pair (kernel launched with clusters of 2)
  bool need_mv = false;  // MV-RNN: U and Mx buffers
  // stats
  int64_t contig = 0, gather = 0, copy_bytes = 0, copy_kernels = 0;
  bool staging = true;      // bf16: stage gathered cell operands into contiguous blocks
  int64_t op_rows = 0;      // staged operand rows appended to H (rows V+1 ..)
  int32_t ext_root_off = 0, num_ext_roots = 0;  // instances whose output is an input lookup
  // largest id read from each weight set's emb / emb2 table (-1: none); ed_execute checks them
  // against emb_rows / emb2_rows, so a bad token fails the call instead of reading out of bounds
  int32_t max_emb[ed::kMaxWeightSets], max_emb2[ed::kMaxWeightSets];
  std::string bad_ext;  // non-empty: an external input where the kernel cannot read one
  int64_t staged = 0, staged_bytes = 0;
  int64_t dst_base = 0;     // idx offset of dst_off[V + 2] (then the copy destinations)
  double plan_us = 0, sched_us = 0, layout_us = 0, validate_us = 0, lower_us = 0;
  // upload state
  std::vector<uint8_t> blob;          // [ts zeros | steps | idx | roots]
  int grid = 0;
  uint32_t launches = 0;
};

// ------------------------------------------------------------------------------------------------
// validation + merge (SURVEY A-5, A-24)
// ------------------------------------------------------------------------------------------------
static ed_status_t validate_and_merge(ed_plan_t *pl, const ed_graph_t *graphs, int32_t ng) {
  const int nt = static_cast<int>(pl->types.size());
  std::fill(pl->max_emb, pl->max_emb + ed::kMaxWeightSets, -1);
  std::fill(pl->max_emb2, pl->max_emb2 + ed::kMaxWeightSets, -1);
  int64_t total = 0;
  for (int gi = 0; gi < ng; ++gi) {
    const ed_graph_t &g = graphs[gi];
    if (g.num_nodes < 0) return fail(ED_E_INVALID_ARG, "graph " + std::to_string(gi) + ": negative num_nodes");
    if (g.num_nodes > 0 && (!g.type || !g.in_off))
      return fail(ED_E_INVALID_ARG, "graph " + std::to_string(gi) + ": null type/in_off");
    total += g.num_nodes;
  }
  if (total >= (int64_t(1) << 30)) return fail(ED_E_INVALID_ARG, "too many nodes");
  {
    int64_t edges = 0;
    for (int gi = 0; gi < ng; ++gi)
      if (graphs[gi].num_nodes > 0) edges += std::max<int64_t>(0, graphs[gi].in_off[graphs[gi].num_nodes]);
    pl->in_idx.reserve(static_cast<size_t>(edges));
  }
  pl->V = total;
  pl->ninst = ng;
  pl->gtype.resize(total);
  pl->in_off.assign(total + 1, 0);
  pl->ext.assign(total, -1);
  pl->roots.resize(ng);
  int64_t base = 0;
  for (int gi = 0; gi < ng; ++gi) {
    const ed_graph_t &g = graphs[gi];
    const std::string tag = "graph " + std::to_string(gi);
    const int n = g.num_nodes;
    if (n > 0 && g.in_off[0] != 0) return fail(ED_E_INVALID_ARG, tag + ": in_off[0] != 0");
    for (int v = 0; v < n; ++v) {
      if (g.in_off[v + 1] < g.in_off[v]) return fail(ED_E_INVALID_ARG, tag + ": in_off not monotone");
      const int t = g.type[v];
      if (t < 0 || t >= nt) return fail(ED_E_TYPE, tag + ": node " + std::to_string(v) + " has unknown type");
      const ed_op_type_t &ot = pl->types[t];
      const int deg = g.in_off[v + 1] - g.in_off[v];
      if (ot.variadic ? deg < ot.num_slots : deg != ot.num_slots)
        return fail(ED_E_ARITY, tag + ": node " + std::to_string(v) + " has " + std::to_string(deg) +
                                    " inputs, type expects " + std::to_string(ot.num_slots));
      if (deg > 0 && !g.in_idx) return fail(ED_E_INVALID_ARG, tag + ": null in_idx");
      for (int k = g.in_off[v]; k < g.in_off[v + 1]; ++k) {
        const int x = g.in_idx[k];
        if (x >= 0) {
          if (x >= n) return fail(ED_E_DANGLING, tag + ": node " + std::to_string(v) + " input " + std::to_string(x) + " out of range");
          if (x == v) return fail(ED_E_CYCLE, tag + ": self loop at node " + std::to_string(v));
          pl->in_idx.push_back(static_cast<int32_t>(base + x));
        } else {
          if (x != ED_ZERO_INPUT) {
            // external (-1 - id): a word row of the op's weight set (TreeFC / MV-RNN children,
            // SURVEY A-6) or the end char x_e of a lattice word (slot 1, read from emb2); any other
            // slot has no table to read it from
            const int j = k - g.in_off[v];
            const bool to_emb = ot.cell_kind == ED_CELL_TREEFC_INTERNAL || ot.cell_kind == ED_CELL_MVRNN_INTERNAL;
            const bool to_emb2 = ot.cell_kind == ED_CELL_LATTICE_WORD && j == 1;
            if (j >= ot.num_slots || !(to_emb || to_emb2)) {
              // a legal dataflow graph for the scheduler, but the kernel has no row to read:
              // planning proceeds, ed_execute refuses the plan
              if (pl->bad_ext.empty())
                pl->bad_ext = tag + ": node " + std::to_string(v) + " slot " + std::to_string(j) +
                              " takes an external input, which this cell cannot read (only TreeFC / MV-RNN"
                              " children and a lattice word's end char are table rows)";
            } else {
              int32_t &mx = to_emb ? pl->max_emb[ot.weight_set] : pl->max_emb2[ot.weight_set];
              mx = std::max(mx, -1 - x);
            }
          }
          pl->in_idx.push_back(x);  // ED_ZERO_INPUT or external (-1 - id)
        }
      }
      pl->gtype[base + v] = t;
      pl->in_off[base + v + 1] = static_cast<int32_t>(pl->in_idx.size());
      if (ot.has_ext) {
        if (!g.ext) return fail(ED_E_INVALID_ARG, tag + ": type with ext but ext == NULL");
        if (g.ext[v] < 0) return fail(ED_E_INVALID_ARG, tag + ": node " + std::to_string(v) + " has no ext token");
        pl->ext[base + v] = g.ext[v];
        pl->max_emb[ot.weight_set] = std::max(pl->max_emb[ot.weight_set], g.ext[v]);
      }
    }
    if (g.root >= n) return fail(ED_E_DANGLING, tag + ": root out of range");
    if (g.root < 0 && n > 0) return fail(ED_E_DANGLING, tag + ": external root on a graph with ops");
    pl->roots[gi] = g.root >= 0 ? static_cast<int32_t>(base + g.root) : g.root;
    if (g.root < 0) {  // a 0-op instance: its output is the input row (-1 - root) of types[0]'s table
      int32_t &mx = pl->max_emb[pl->types[0].weight_set];
      mx = std::max(mx, -1 - g.root);
    }
    base += n;
  }
  // acyclicity (Kahn); the consumers CSR and in-degrees are kept for Alg. 1
  std::vector<int32_t> &indeg = pl->indeg;
  std::vector<int32_t> &coff = pl->coff;
  indeg.assign(total, 0);
  coff.assign(total + 1, 0);
  for (int64_t v = 0; v < total; ++v)
    for (int k = pl->in_off[v]; k < pl->in_off[v + 1]; ++k)
      if (pl->in_idx[k] >= 0) { ++indeg[v]; ++coff[pl->in_idx[k] + 1]; }
  for (int64_t v = 0; v < total; ++v) coff[v + 1] += coff[v];
  std::vector<int32_t> &cons = pl->cons;
  cons.assign(coff[total], 0);
  {
    std::vector<int32_t> fill(coff.begin(), coff.end() - 1);
    for (int64_t v = 0; v < total; ++v)
      for (int k = pl->in_off[v]; k < pl->in_off[v + 1]; ++k)
        if (pl->in_idx[k] >= 0) cons[fill[pl->in_idx[k]]++] = static_cast<int32_t>(v);
  }
  std::vector<int32_t> stack;
  for (int64_t v = 0; v < total; ++v)
    if (indeg[v] == 0) stack.push_back(static_cast<int32_t>(v));
  int64_t seen = 0;
  std::vector<int32_t> d = indeg;
  while (!stack.empty()) {
    const int32_t v = stack.back();
    stack.pop_back();
    ++seen;
    for (int k = coff[v]; k < coff[v + 1]; ++k)
      if (--d[cons[k]] == 0) stack.push_back(cons[k]);
  }
  if (seen != total) return fail(ED_E_CYCLE, "dataflow graph has a cycle");
  return ED_OK;
}

// ------------------------------------------------------------------------------------------------
// Alg. 1 with E_sort / E_base + table lookup; fallback key[0] (A-3)
// ------------------------------------------------------------------------------------------------
// Ascending sort of node ids (< 2^30): LSD radix (3 x 10-bit digits) for large batches, std::sort
// for small ones.
static void sort_ids(std::vector<int32_t> *v, std::vector<int32_t> *tmp) {
  const size_t n = v->size();
  if (n < 2048) {
    std::sort(v->begin(), v->end());
    return;
  }
  tmp->resize(n);
  int32_t *a = v->data(), *b = tmp->data();
  for (int shift = 0; shift < 30; shift += 10) {
    uint32_t cnt[1025] = {0};
    for (size_t i = 0; i < n; ++i) ++cnt[((static_cast<uint32_t>(a[i]) >> shift) & 1023u) + 1];
    for (int d = 0; d < 1024; ++d) cnt[d + 1] += cnt[d];
    for (size_t i = 0; i < n; ++i) b[cnt[(static_cast<uint32_t>(a[i]) >> shift) & 1023u]++] = a[i];
    std::swap(a, b);
  }
  if (a != v->data()) std::copy(a, a + n, v->data());
}

static ed_status_t schedule(ed_plan_t *pl, const ed_fsm_t *fsm, int policy) {
  std::vector<int32_t> sort_tmp;
  const int nt = static_cast<int>(pl->types.size());
  const int64_t V = pl->V;
  // comparators: topological depth (1 + max over node inputs; raw inputs 0)
  std::vector<int32_t> depth;
  std::vector<double> mean_depth;
  std::vector<int32_t> sc_seq;
  if (policy == ED_POLICY_DEPTH || policy == ED_POLICY_AGENDA) {
    depth.assign(V, 0);
    std::vector<int32_t> d(pl->indeg), q;
    q.reserve(V);
    for (int64_t v = 0; v < V; ++v)
      if (d[v] == 0) q.push_back(static_cast<int32_t>(v));
    for (size_t hh = 0; hh < q.size(); ++hh) {
      const int32_t v = q[hh];
      int32_t dv = 0;
      for (int k = pl->in_off[v]; k < pl->in_off[v + 1]; ++k)
        if (pl->in_idx[k] >= 0) dv = std::max(dv, depth[pl->in_idx[k]]);
      depth[v] = dv + 1;
      for (int k = pl->coff[v]; k < pl->coff[v + 1]; ++k)
        if (--d[pl->cons[k]] == 0) q.push_back(pl->cons[k]);
    }
  }
  if (policy == ED_POLICY_AGENDA) {  // mean depth over all nodes of the type (A-22)
    std::vector<int64_t> sum(nt, 0), cnt(nt, 0);
    for (int64_t v = 0; v < V; ++v) {
      sum[pl->gtype[v]] += depth[v];
      ++cnt[pl->gtype[v]];
    }
    mean_depth.assign(nt, std::numeric_limits<double>::infinity());
    for (int t = 0; t < nt; ++t)
      if (cnt[t]) mean_depth[t] = static_cast<double>(sum[t]) / static_cast<double>(cnt[t]);
  }
  if (policy == ED_POLICY_SC) {  // the type sequence of the SC chooser on the merged graph
    ed::RlGraph g;
    g.n = static_cast<int32_t>(V);
    g.type = pl->gtype;
    g.pred_off.assign(1, 0);
    for (int64_t v = 0; v < V; ++v) {
      std::vector<int32_t> pr;
      for (int k = pl->in_off[v]; k < pl->in_off[v + 1]; ++k)
        if (pl->in_idx[k] >= 0) pr.push_back(pl->in_idx[k]);
      std::sort(pr.begin(), pr.end());
      pr.erase(std::unique(pr.begin(), pr.end()), pr.end());
      g.preds.insert(g.preds.end(), pr.begin(), pr.end());
      g.pred_off.push_back(static_cast<int32_t>(g.preds.size()));
    }
    sc_seq = ed::sc_type_sequence(g, nt);
  }
  std::map<std::vector<int32_t>, int32_t> table;
  int encoder = ED_ENC_SORT;
  if (fsm) {
    encoder = fsm->encoder;
    if (encoder != ED_ENC_SORT && encoder != ED_ENC_BASE && encoder != ED_ENC_MAX) return fail(ED_E_FSM, "unknown encoder");
    if (fsm->fallback != ED_FALLBACK_KEY0) return fail(ED_E_FSM, "unknown fallback");
    if (fsm->num_entries > 0 && !fsm->entries) return fail(ED_E_FSM, "null entries");
    for (int e = 0; e < fsm->num_entries; ++e) {
      const ed_fsm_entry_t &en = fsm->entries[e];
      const int set_len = encoder == ED_ENC_MAX ? en.key_len - 1 : en.key_len;  // E_max: set + argmax type
      if (set_len <= 0 || set_len > nt || !en.key) return fail(ED_E_FSM, "entry " + std::to_string(e) + ": bad key");
      std::vector<int32_t> key(en.key, en.key + set_len);
      if (encoder == ED_ENC_MAX) {
        if (!std::is_sorted(key.begin(), key.end()) || std::find(key.begin(), key.end(), en.key[set_len]) == key.end())
          return fail(ED_E_FSM, "entry " + std::to_string(e) + ": E_max key must be an ascending set followed by one of its types");
      }
      std::vector<int32_t> sorted_key = key;
      std::sort(sorted_key.begin(), sorted_key.end());
      for (int k = 0; k < set_len; ++k) {
        if (key[k] < 0 || key[k] >= nt) return fail(ED_E_FSM, "entry " + std::to_string(e) + ": key type out of range");
        if (k > 0 && sorted_key[k] == sorted_key[k - 1]) return fail(ED_E_FSM, "entry " + std::to_string(e) + ": repeated type in key");
      }
      if (std::find(key.begin(), key.end(), en.action) == key.end())
        return fail(ED_E_FSM, "entry " + std::to_string(e) + ": action not present in its key");
      if (encoder == ED_ENC_MAX) key.push_back(en.key[set_len]);
      table[key] = en.action;
    }
  }
  // consumers CSR and remaining-input counters (one count per node-input edge), from validation
  std::vector<int32_t> remaining(pl->indeg);
  const std::vector<int32_t> &coff = pl->coff, &cons = pl->cons;
  std::vector<std::vector<int32_t>> ready(nt);
  for (int64_t v = 0; v < V; ++v)
    if (remaining[v] == 0) ready[pl->gtype[v]].push_back(static_cast<int32_t>(v));
  pl->batch_type.clear();
  pl->batch_off.assign(1, 0);
  pl->members.clear();
  pl->members.reserve(V);
  std::vector<int32_t> key, order(nt);
  int64_t done = policy == ED_POLICY_DEPTH ? V : 0;  // depth-based: grouped below, no Alg. 1
  while (done < V) {
    key.clear();
    for (int t = 0; t < nt; ++t)
      if (!ready[t].empty()) key.push_back(t);
    if (key.empty()) return fail(ED_E_CYCLE, "no ready node (internal)");
    std::vector<int32_t> skey = key;  // E_sort: descending count, ties ascending id
    std::stable_sort(skey.begin(), skey.end(), [&](int a, int b) { return ready[a].size() > ready[b].size(); });
    std::vector<int32_t> mkey;
    if (encoder == ED_ENC_MAX) {  // (E_base, most frequent type) = ascending set + skey[0]
      mkey = key;
      mkey.push_back(skey[0]);
    }
    const std::vector<int32_t> &lookup = encoder == ED_ENC_SORT ? skey : (encoder == ED_ENC_MAX ? mkey : key);
    int32_t act = -1;
    if (policy == ED_POLICY_FSM) {
      auto it = table.find(lookup);
      if (it != table.end()) act = it->second;
    } else if (policy == ED_POLICY_AGENDA) {
      for (int t : key)
        if (act < 0 || mean_depth[t] < mean_depth[act]) act = t;
    } else if (policy == ED_POLICY_SC) {
      act = sc_seq[pl->batch_type.size()];
    }
    if (act < 0 || ready[act].empty()) act = skey[0];
    std::vector<int32_t> batch;
    batch.swap(ready[act]);
    sort_ids(&batch, &sort_tmp);
    for (int32_t v : batch) {
      pl->members.push_back(v);
      for (int k = coff[v]; k < coff[v + 1]; ++k) {
        const int32_t w = cons[k];
        if (--remaining[w] == 0) ready[pl->gtype[w]].push_back(w);
      }
    }
    done += static_cast<int64_t>(batch.size());
    pl->batch_type.push_back(act);
    pl->batch_off.push_back(static_cast<int32_t>(pl->members.size()));
  }
  if (policy == ED_POLICY_DEPTH) {  // TF-Fold: one batch per (depth, type), ascending
    std::vector<int64_t> keyv(V);
    std::vector<int32_t> ord(V);
    for (int64_t v = 0; v < V; ++v) {
      keyv[v] = static_cast<int64_t>(depth[v]) * nt + pl->gtype[v];
      ord[v] = static_cast<int32_t>(v);
    }
    std::stable_sort(ord.begin(), ord.end(), [&](int32_t a, int32_t b) { return keyv[a] < keyv[b]; });
    pl->batch_type.clear();
    pl->batch_off.assign(1, 0);
    pl->members.assign(ord.begin(), ord.end());
    for (int64_t k = 0; k < V; ++k)
      if (k + 1 == V || keyv[ord[k + 1]] != keyv[ord[k]]) {
        pl->batch_type.push_back(pl->gtype[ord[k]]);
        pl->batch_off.push_back(static_cast<int32_t>(k + 1));
      }
  }
  // App. B.3 lower bound: per type, the max number of type-t nodes on a path (= Depth(G^t)).
  // one pass over the schedule order (a topological order) with nt counters per node
  int64_t lb = 0;
  std::vector<int32_t> cnt(static_cast<size_t>(V) * nt, 0), best(nt, 0), c(nt);
  for (int32_t v : pl->members) {
    std::fill(c.begin(), c.end(), 0);
    for (int k = pl->in_off[v]; k < pl->in_off[v + 1]; ++k)
      if (pl->in_idx[k] >= 0) {
        const int32_t *cu = &cnt[static_cast<size_t>(pl->in_idx[k]) * nt];
        for (int t = 0; t < nt; ++t) c[t] = std::max(c[t], cu[t]);
      }
    int32_t *cv = &cnt[static_cast<size_t>(v) * nt];
    for (int t = 0; t < nt; ++t) {
      cv[t] = c[t] + (pl->gtype[v] == t ? 1 : 0);
      best[t] = std::max(best[t], cv[t]);
    }
  }
  for (int t = 0; t < nt; ++t) lb += best[t];
  pl->lower_bound = lb;
  return ED_OK;
}

// ------------------------------------------------------------------------------------------------
// lowering: node rows -> device step table
// ------------------------------------------------------------------------------------------------
// Split-K over CTA pairs; ED_SPLIT=0 turns it off (A/B development switch).
static bool split_enabled() {
  const char *v = std::getenv("ED_SPLIT");  // read per plan (tests switch it)
  return !(v && std::atoi(v) == 0);
}

static ed_status_t lower(ed_plan_t *pl) {
  const int64_t V = pl->V;
  const int zero_row = static_cast<int32_t>(V);
  const int nb = static_cast<int>(pl->batch_type.size());
  const int h = pl->hidden;
  pl->idx.clear();
  pl->slot_modes.assign(static_cast<size_t>(nb) * 2, -1);
  pl->contig = pl->gather = pl->copy_bytes = pl->copy_kernels = 0;
  const int64_t row_bytes = static_cast<int64_t>(h) * (pl->dtype == ED_BF16 ? 2 : 4);
  auto encode = [&](int32_t x) -> int32_t {
    if (x >= 0) return pl->row_of_node[x];
    if (x == ED_ZERO_INPUT) return zero_row;
    return x;  // external id
  };
  pl->steps.clear();
  pl->has_split = false;
  pl->op_rows = pl->staged = pl->staged_bytes = 0;
  std::vector<std::pair<int32_t, int32_t>> stage_pairs;  // (producer row, staged H row)
  const bool staging = pl->staging && pl->dtype == ED_BF16;
  // device order of the batches: stable by dependency level (ED_ORDER_LEVEL), else schedule order
  std::vector<int32_t> border(nb);
  for (int b = 0; b < nb; ++b) border[b] = b;
  if (pl->level_order) {
    std::vector<int32_t> batch_of(V, -1), level(nb, 0);
    for (int b = 0; b < nb; ++b)
      for (int k = pl->batch_off[b]; k < pl->batch_off[b + 1]; ++k) batch_of[pl->members[k]] = b;
    for (int b = 0; b < nb; ++b) {
      int32_t lv = 0;
      for (int k = pl->batch_off[b]; k < pl->batch_off[b + 1]; ++k) {
        const int32_t v = pl->members[k];
        for (int q = pl->in_off[v]; q < pl->in_off[v + 1]; ++q)
          if (pl->in_idx[q] >= 0) lv = std::max(lv, level[batch_of[pl->in_idx[q]]] + 1);
      }
      level[b] = lv;
    }
    std::stable_sort(border.begin(), border.end(), [&](int32_t a, int32_t c) { return level[a] < level[c]; });
  }
  pl->step_batch.clear();
  for (int bi = 0; bi < nb; ++bi) {
    const int b = border[bi];
    const int t = pl->batch_type[b];
    const ed_op_type_t &ot = pl->types[t];
    // members in result-row order: a batch's rows are one block (A-9), so each member goes to
    // position row - min row directly (no comparison sort); a non-block result fails below
    const int m = pl->batch_off[b + 1] - pl->batch_off[b];
    std::vector<int32_t> mem(m, -1);
    {
      int32_t rmin = INT32_MAX;
      for (int k = pl->batch_off[b]; k < pl->batch_off[b + 1]; ++k) rmin = std::min(rmin, pl->row_of_node[pl->members[k]]);
      for (int k = pl->batch_off[b]; k < pl->batch_off[b + 1]; ++k) {
        const int32_t v = pl->members[k], pos = pl->row_of_node[v] - rmin;
        if (pos < 0 || pos >= m || mem[pos] != -1)
          return fail(ED_E_INVALID_ARG, "internal: result operand of batch " + std::to_string(b) + " not contiguous");
        mem[pos] = v;
      }
    }
    std::copy(mem.begin(), mem.end(), pl->members.begin() + pl->batch_off[b]);
    ed::DevStep st{};
    st.cell = ot.cell_kind;
    st.m = m;
    st.out_row0 = pl->row_of_node[mem[0]];
    for (int i = 0; i < m; ++i)
      if (pl->row_of_node[mem[i]] != st.out_row0 + i)
        return fail(ED_E_INVALID_ARG, "internal: result operand of batch " + std::to_string(b) + " not contiguous");
    st.wset = ot.weight_set;
    st.ext_off = -1;
    st.var_off = -1;
    st.gates = ot.cell_kind == ED_CELL_LINEAR_OUT ? ot.out_dim : ed::cell_gates(ot.cell_kind);
    st.units = ed::cell_units(ot.cell_kind);
    if (st.units > 0 && pl->dtype == ED_BF16) {
      // narrower column tiles for small batches: the fewest units per tile (multiple of 16, <= the
      // cell's maximum) whose tile count still fits one wave of 148 CTAs; a tile's time is set by
      // its K-chunk chain (operand gather), so more concurrent tiles = shorter batch
      const int mt = (m + 127) / 128;
      const int umax = st.units;
      for (int u = umax; u >= 16; u -= 16)
        if (mt * ((h + u - 1) / u) <= 148) st.units = u;
      // development override for batches that do not fit one wave: ED_UNITS="cell:units,..."
      // (scripts/units_sweep.sh)
      static const char *ov = std::getenv("ED_UNITS");
      if (ov && mt * ((h + st.units - 1) / st.units) > 148) {
        for (const char *q = ov; *q;) {
          int c = 0, u = 0, n = 0;
          if (std::sscanf(q, "%d:%d%n", &c, &u, &n) != 2) break;
          if (c == ot.cell_kind && u >= 16 && u <= umax && u % 16 == 0) st.units = u;
          q += n;
          if (*q == ',') ++q;
        }
      }
    }
    st.n_col_tiles = st.units > 0 ? (h + st.units - 1) / st.units : 0;
    if (pl->dtype == ED_BF16 && st.units == 16 && h % 16 == 0 && ed::cell_splittable(ot.cell_kind) &&
        (ed::cell_segments(ot.cell_kind) * h / 64) % 2 == 0 &&
        2 * ((m + 127) / 128) * st.n_col_tiles <= 148 && split_enabled()) {
      // split-K over a CTA pair (cluster of 2) for batches of at most half a wave of 16-unit tiles:
      // each CTA streams half of the tile's K (half its operand and weight bytes, half the MMA
      // chain) and runs the gate epilogue of one 8-unit half after a DSMEM exchange of partials
      st.wsel |= ed::kStepSplitK;
      pl->has_split = true;
    }
    if (ot.cell_kind == ED_CELL_LINEAR_OUT && pl->dtype == ED_BF16) {
      // bf16 output linear on the tensor cores: one N = 16 column tile (C <= 16 classes, rows >= C
      // of the packed W_O are zero); units = C, gates = 1
      st.gates = 1;
      st.units = ot.out_dim;
      st.n_col_tiles = 1;
    }
    st.nslots = std::min(ot.num_slots, ed::kMaxSlotsDev);
    std::vector<int32_t> slot_entries[ed::kMaxSlotsDev];
    for (int j = 0; j < st.nslots; ++j) {
      std::vector<int32_t> &ent = slot_entries[j];
      ent.resize(m);
      bool contig = true;
      for (int i = 0; i < m; ++i) {
        ent[i] = encode(pl->in_idx[pl->in_off[mem[i]] + j]);
        const int32_t raw = pl->in_idx[pl->in_off[mem[i]] + j];
        if (raw < 0 || ent[i] != ent[0] + i) contig = false;
      }
      if (contig) {
        st.mode[j] = 1;
        st.arg[j] = ent[0];
        ++pl->contig;
      } else {
        st.mode[j] = 0;
        st.arg[j] = static_cast<int32_t>(pl->idx.size());
        pl->idx.insert(pl->idx.end(), ent.begin(), ent.end());
        ++pl->gather;
        pl->copy_bytes += 2 * static_cast<int64_t>(m) * row_bytes;
        ++pl->copy_kernels;
        // Staging (bf16 tensor-core cells whose slot j is an A operand, batches of >= 128 members
        // where the loaders use 128-row TMA boxes): if every entry is a produced row (or the zero
        // state), the batch gets a block of m H rows after the node records; each producer's
        // epilogue also stores its h row there, and the loaders read the block as TMA boxes
        // instead of gathering 16 B pieces of m scattered rows (~25 GB/s per SM on B200).
        const bool a_operand = ed::cell_gates(ot.cell_kind) > 0 && ot.cell_kind != ED_CELL_MVRNN_INTERNAL &&
                               !(ot.cell_kind == ED_CELL_LATTICE_WORD && j == 1);
        bool ok = staging && a_operand && m >= 128;
        for (int i = 0; i < m && ok; ++i) {
          const int32_t raw = pl->in_idx[pl->in_off[mem[i]] + j];
          ok = raw >= 0 || raw == ED_ZERO_INPUT;
        }
        if (ok) {
          const int32_t base = static_cast<int32_t>(V + 1 + pl->op_rows);
          pl->idx.push_back(base);
          for (int i = 0; i < m; ++i)
            if (ent[i] != zero_row) stage_pairs.emplace_back(ent[i], base + i);
          pl->op_rows += m;
          ++pl->staged;
          pl->staged_bytes += static_cast<int64_t>(m) * row_bytes;
          st.mode[j] = 2;
        }
      }
      pl->slot_modes[static_cast<size_t>(b) * 2 + j] = st.mode[j] == 1 ? 1 : 0;
    }
    if (ot.has_ext) {
      st.ext_off = static_cast<int32_t>(pl->idx.size());
      for (int i = 0; i < m; ++i) pl->idx.push_back(pl->ext[mem[i]]);
    }
    if (ot.variadic) {
      st.var_off = static_cast<int32_t>(pl->idx.size());
      const size_t offs = pl->idx.size();
      pl->idx.resize(offs + m + 1);
      for (int i = 0; i < m; ++i) {
        pl->idx[offs + i] = static_cast<int32_t>(pl->idx.size());
        for (int k = pl->in_off[mem[i]] + ot.num_slots; k < pl->in_off[mem[i] + 1]; ++k)
          pl->idx.push_back(encode(pl->in_idx[k]));
      }
      pl->idx[offs + m] = static_cast<int32_t>(pl->idx.size());
    }
    pl->steps.push_back(st);
    pl->step_batch.push_back(b);
    // two-contraction cells: the dependent second GEMM is its own device step over the same rows
    if (ot.cell_kind == ED_CELL_LATTICE_WORD) {
      ed::DevStep s2 = st;  // l = s(W_l [x_e; c^w] + b_l): x_e = slot 1 (external char), c^w = own row
      s2.cell = ed::kCellLatticeLink;
      s2.wsel = 1;
      s2.ext_off = -1;
      s2.gates = 1;
      s2.units = ed::cell_units(s2.cell);
      s2.n_col_tiles = (h + s2.units - 1) / s2.units;
      s2.mode[0] = st.mode[1];
      s2.arg[0] = st.arg[1];
      s2.mode[1] = 1;
      s2.arg[1] = st.out_row0;
      s2.nslots = 2;
      pl->steps.push_back(s2);
      pl->step_batch.push_back(b);
    } else if (ot.cell_kind == ED_CELL_MVRNN_INTERNAL) {
      // step 1 (st): u = [B a; A b] (SIMT matvecs) -> U; step 2: p = tanh(W u + b) -> H, reading the
      // node's own U rows; step 3: P^T = [A^T | B^T] W_M^T -> Mx (rows m*h, K = 2h, N = h)
      pl->steps.back().units = 0;
      pl->steps.back().n_col_tiles = 0;
      ed::DevStep sp = st;
      sp.cell = ed::kCellMvP;
      sp.wsel = 0;
      sp.gates = 1;
      sp.units = ed::cell_units(sp.cell);
      if (pl->dtype == ED_BF16) {
        const int mt = (m + 127) / 128;
        for (int u = sp.units; u >= 16; u -= 16)
          if (mt * ((h + u - 1) / u) <= 148) sp.units = u;
      }
      sp.n_col_tiles = (h + sp.units - 1) / sp.units;
      sp.mode[0] = 1;
      sp.arg[0] = st.out_row0;
      sp.mode[1] = 0;
      sp.arg[1] = 0;
      sp.nslots = 1;
      pl->steps.push_back(sp);
      pl->step_batch.push_back(b);
      ed::DevStep sm = st;
      sm.cell = ed::kCellMvMat;
      sm.wsel = 1;
      sm.gates = 1;
      sm.units = ed::cell_units(sm.cell);
      if (pl->dtype == ED_BF16) {
        const int64_t mt = (static_cast<int64_t>(m) * h + 127) / 128;
        for (int u = sm.units; u >= 16; u -= 16)
          if (mt * ((h + u - 1) / u) <= 148) sm.units = u;
      }
      sm.n_col_tiles = (h + sm.units - 1) / sm.units;
      pl->steps.push_back(sm);
      pl->step_batch.push_back(b);
    } else if (ot.cell_kind == ED_CELL_TAGGER) {
      ed::DevStep s2 = st;  // y = W2 t + b2 with t in the node's own h row
      s2.cell = ed::kCellTaggerOut;
      s2.wsel = 1;
      s2.gates = ot.out_dim;
      s2.units = 0;
      s2.n_col_tiles = 0;
      s2.mode[0] = 1;
      s2.arg[0] = st.out_row0;
      s2.nslots = 1;
      pl->steps.push_back(s2);
      pl->step_batch.push_back(b);
    }
  }
  // instance outputs: the epilogue producing an instance's root row also stores it into
  // out_root[instance] (a copy entry -1 - instance); roots that are input lookups are copied by CTA 0
  std::vector<int32_t> ext_roots;
  for (int i = 0; i < pl->ninst; ++i) {
    const int32_t r = pl->roots[i];
    if (r >= 0)
      stage_pairs.emplace_back(pl->row_of_node[r], -1 - i);
    else {
      ext_roots.push_back(i);
      ext_roots.push_back(-1 - r);
    }
  }
  pl->ext_root_off = static_cast<int32_t>(pl->idx.size());
  pl->num_ext_roots = static_cast<int32_t>(ext_roots.size() / 2);
  pl->idx.insert(pl->idx.end(), ext_roots.begin(), ext_roots.end());
  // copies of every result row into staged operand blocks and instance outputs (CSR over rows
  // 0..V), appended to idx
  {
    std::vector<int32_t> cnt(V + 2, 0);
    for (const auto &pr : stage_pairs) ++cnt[pr.first + 1];
    for (int64_t r = 0; r <= V; ++r) cnt[r + 1] += cnt[r];
    pl->dst_base = static_cast<int64_t>(pl->idx.size());
    const int32_t base2 = static_cast<int32_t>(pl->dst_base + V + 2);
    for (int64_t r = 0; r <= V + 1; ++r) pl->idx.push_back(base2 + cnt[r]);
    pl->idx.resize(pl->idx.size() + stage_pairs.size());
    std::vector<int32_t> fill(cnt.begin(), cnt.end() - 1);
    for (const auto &pr : stage_pairs) pl->idx[base2 + fill[pr.first]++] = pr.second;
  }
  // readiness: target[row] = sum of what every device step writing the row publishes; a step that
  // reads its own rows waits for what the earlier steps of its batch publish (self_need)
  pl->target.assign(V + 1, 0);
  for (size_t k = 0; k < pl->steps.size(); ++k) {
    ed::DevStep &st = pl->steps[k];
    st.self_need = 0;
    for (size_t q = k; q-- > 0 && pl->steps[q].out_row0 == st.out_row0 && pl->steps[q].m == st.m;)
      st.self_need += ed::step_contrib(pl->steps[q].cell, h);
    for (int i = 0; i < st.m; ++i) pl->target[st.out_row0 + i] += ed::step_contrib(st.cell, h);
  }
  pl->root_rows.resize(pl->ninst);
  for (int i = 0; i < pl->ninst; ++i) {
    const int32_t r = pl->roots[i];
    pl->root_rows[i] = r >= 0 ? pl->row_of_node[r] : r;
  }
  // workspace layout
  const int64_t rows = V + 1;
  const size_t elt = pl->dtype == ED_BF16 ? 2 : 4;
  size_t off = 0;
  pl->off_bar = off; off += 256;  // header: binding nonce (8 B)
  const size_t nsteps = pl->steps.size();
  pl->off_ts = off; off = align_up(off + 8 * (nsteps + 1), 256);
  pl->off_steps = off; off = align_up(off + sizeof(ed::DevStep) * nsteps, 256);
  pl->off_idx = off; off = align_up(off + 4 * pl->idx.size(), 256);
  pl->off_roots = off; off = align_up(off + 4 * static_cast<size_t>(pl->ninst), 256);
  pl->off_target = off; off = align_up(off + 4 * static_cast<size_t>(rows), 256);
  pl->off_ready = off; off = align_up(off + 4 * static_cast<size_t>(rows), 1024);
  pl->off_h = off; off = align_up(off + elt * (rows + pl->op_rows) * h, 1024);
  pl->off_c = off; off = align_up(off + 4 * rows * h, 1024);
  pl->y_cols = 0;
  pl->need_x = false;
  for (const auto &ot : pl->types) {
    if (ot.cell_kind == ED_CELL_LINEAR_OUT || ot.cell_kind == ED_CELL_TAGGER)
      pl->y_cols = std::max<int64_t>(pl->y_cols, ot.out_dim);
    if (ot.cell_kind == ED_CELL_LATTICE_WORD) pl->need_x = true;
  }
  pl->need_mv = false;
  for (const auto &ot : pl->types)
    if (ot.cell_kind == ED_CELL_MVRNN_INTERNAL) pl->need_mv = true;
  pl->off_y = off; off = align_up(off + 4 * rows * pl->y_cols, 1024);
  pl->off_x = off; if (pl->need_x) off = align_up(off + 4 * rows * h, 1024);
  pl->off_u = off; if (pl->need_mv) off = align_up(off + elt * rows * 2 * h, 1024);
  pl->off_m = off; if (pl->need_mv) off = align_up(off + elt * rows * h * h, 1024);
  pl->ws_bytes = off;
  // host blob mirrors [header .. target] so one async H2D uploads the static part (the header's
  // nonce is filled in per binding)
  pl->blob.assign(pl->off_ready - pl->off_bar, 0);
  std::memcpy(pl->blob.data() + (pl->off_steps - pl->off_bar), pl->steps.data(), sizeof(ed::DevStep) * nsteps);
  if (!pl->idx.empty()) std::memcpy(pl->blob.data() + (pl->off_idx - pl->off_bar), pl->idx.data(), 4 * pl->idx.size());
  if (pl->ninst) std::memcpy(pl->blob.data() + (pl->off_roots - pl->off_bar), pl->root_rows.data(), 4 * pl->ninst);
  std::memcpy(pl->blob.data() + (pl->off_target - pl->off_bar), pl->target.data(), 4 * pl->target.size());
  return ED_OK;
}

// ------------------------------------------------------------------------------------------------
// ABI
// ------------------------------------------------------------------------------------------------
extern "C" {

const char *ed_last_error(void) { return g_last_error.c_str(); }

// ------------------------------------------------------------------------------------------------
// FSM learning (PAPER §2.3): graphs validated as for ed_plan, split back into instances
// ------------------------------------------------------------------------------------------------
struct ed_fsm_learned_s {
  ed::RlResult res;
  int32_t encoder = ED_ENC_SORT;
  std::vector<std::vector<int32_t>> keys;   // table keys (storage for the ed_fsm_t view)
  std::vector<ed_fsm_entry_t> entries;
  std::vector<std::pair<std::vector<int32_t>, std::pair<int32_t, double>>> qlist;
  double learn_us = 0;
};

ed_status_t ed_fsm_learn(const ed_graph_t *graphs, int32_t num_graphs, const ed_op_type_t *types, int32_t num_types,
                         const ed_rl_config_t *cfg, ed_fsm_learned_t **out) {
  const double t0 = now_us();
  if (!out || !cfg) return fail(ED_E_INVALID_ARG, "null argument");
  *out = nullptr;
  if (num_graphs <= 0 || !graphs) return fail(ED_E_INVALID_ARG, "no graphs");
  if (num_types <= 0 || !types) return fail(ED_E_INVALID_ARG, "bad types");
  ed_plan_t tmp;
  tmp.types.assign(types, types + num_types);
  ed_status_t st = validate_and_merge(&tmp, graphs, num_graphs);
  if (st != ED_OK) return st;
  // Episode graphs: each instance with local ids, or (ED_RL_EPISODE_MERGED) the merged minibatch
  // with its global ids (one graph: the dataflow graph ed_plan schedules).
  const bool merged = cfg->episode_graph == ED_RL_EPISODE_MERGED;
  std::vector<ed::RlGraph> gs(merged ? 1 : num_graphs);
  int64_t base = 0;
  for (int gi = 0; gi < num_graphs; ++gi) {
    ed::RlGraph &g = gs[merged ? 0 : gi];
    const int64_t off = merged ? 0 : base;  // id offset of this graph's first node in g
    if (g.pred_off.empty()) g.pred_off.assign(1, 0);
    const int32_t n = graphs[gi].num_nodes;
    g.type.insert(g.type.end(), tmp.gtype.begin() + base, tmp.gtype.begin() + base + n);
    for (int v = 0; v < n; ++v) {
      std::vector<int32_t> pr;
      for (int k = tmp.in_off[base + v]; k < tmp.in_off[base + v + 1]; ++k)
        if (tmp.in_idx[k] >= 0) pr.push_back(static_cast<int32_t>(tmp.in_idx[k] - off));
      std::sort(pr.begin(), pr.end());
      pr.erase(std::unique(pr.begin(), pr.end()), pr.end());  // distinct dependencies
      g.preds.insert(g.preds.end(), pr.begin(), pr.end());
      g.pred_off.push_back(static_cast<int32_t>(g.preds.size()));
    }
    g.n += n;
    base += n;
  }
  ed_fsm_learned_t *fl = new (std::nothrow) ed_fsm_learned_t();
  if (!fl) return fail(ED_E_OOM, "out of host memory");
  if (ed::rl_train(gs, num_types, *cfg, &fl->res) != 0) {
    delete fl;
    return fail(ED_E_INVALID_ARG, "bad RL config");
  }
  fl->encoder = cfg->encoder;
  for (const auto &kv : fl->res.table) fl->keys.push_back(kv.first);
  size_t k = 0;
  for (const auto &kv : fl->res.table) {
    fl->entries.push_back(ed_fsm_entry_t{static_cast<int32_t>(fl->keys[k].size()), fl->keys[k].data(), kv.second});
    ++k;
  }
  for (const auto &kv : fl->res.q) fl->qlist.push_back({kv.first.first, {kv.first.second, kv.second}});
  fl->learn_us = now_us() - t0;
  *out = fl;
  return ED_OK;
}

ed_status_t ed_fsm_learned_info(const ed_fsm_learned_t *fl, ed_fsm_learned_info_t *o) {
  if (!fl || !o) return fail(ED_E_INVALID_ARG, "null argument");
  o->episodes = fl->res.episodes;
  o->table_entries = static_cast<int64_t>(fl->entries.size());
  o->q_entries = static_cast<int64_t>(fl->qlist.size());
  o->checkpoints = static_cast<int64_t>(fl->res.checkpoints.size());
  o->final_batches = fl->res.final_batches;
  o->lower_bound = fl->res.lower_bound;
  o->learn_us = fl->learn_us;
  return ED_OK;
}

ed_status_t ed_fsm_learned_table(const ed_fsm_learned_t *fl, ed_fsm_t *o) {
  if (!fl || !o) return fail(ED_E_INVALID_ARG, "null argument");
  o->encoder = fl->encoder;
  o->num_entries = static_cast<int32_t>(fl->entries.size());
  o->entries = fl->entries.empty() ? nullptr : fl->entries.data();
  o->fallback = ED_FALLBACK_KEY0;
  return ED_OK;
}

ed_status_t ed_fsm_learned_q(const ed_fsm_learned_t *fl, int64_t k, int32_t *key, int32_t *key_len, int32_t *action,
                             double *q) {
  if (!fl || !key || !key_len || !action || !q) return fail(ED_E_INVALID_ARG, "null argument");
  if (k < 0 || k >= static_cast<int64_t>(fl->qlist.size())) return fail(ED_E_INVALID_ARG, "entry out of range");
  const auto &e = fl->qlist[k];
  std::copy(e.first.begin(), e.first.end(), key);
  *key_len = static_cast<int32_t>(e.first.size());
  *action = e.second.first;
  *q = e.second.second;
  return ED_OK;
}

ed_status_t ed_fsm_learned_checkpoint(const ed_fsm_learned_t *fl, int64_t c, int64_t *episode, int64_t *batches) {
  if (!fl || !episode || !batches) return fail(ED_E_INVALID_ARG, "null argument");
  if (c < 0 || c >= static_cast<int64_t>(fl->res.checkpoints.size())) return fail(ED_E_INVALID_ARG, "checkpoint out of range");
  *episode = fl->res.checkpoints[c].first;
  *batches = fl->res.checkpoints[c].second;
  return ED_OK;
}

void ed_fsm_learned_destroy(ed_fsm_learned_t *fl) { delete fl; }

const char *ed_version(void) { return "ed_batch 0.1 sm_100a"; }

ed_status_t ed_plan(const ed_graph_t *graphs, int32_t num_graphs, const ed_op_type_t *types, int32_t num_types,
                    const ed_fsm_t *fsm, const ed_plan_opts_t *opts, ed_plan_t **out) {
  const double t0 = now_us();
  if (!out) return fail(ED_E_INVALID_ARG, "out == NULL");
  *out = nullptr;
  if (num_graphs < 0 || (num_graphs > 0 && !graphs)) return fail(ED_E_INVALID_ARG, "bad graphs");
  if (num_types <= 0 || !types) return fail(ED_E_INVALID_ARG, "bad types");
  const int layout = opts ? opts->layout : ED_LAYOUT_SCHEDULE_ORDER;
  if (layout != ED_LAYOUT_SCHEDULE_ORDER && layout != ED_LAYOUT_PQ) return fail(ED_E_INVALID_ARG, "unknown layout");
  if (opts)
    for (int k = 0; k < 4; ++k)
      if (opts->reserved[k] != 0) return fail(ED_E_INVALID_ARG, "opts.reserved must be 0");
  if (opts && opts->step_order != ED_ORDER_LEVEL && opts->step_order != ED_ORDER_SCHEDULE)
    return fail(ED_E_INVALID_ARG, "unknown step order");
  if (opts && (opts->policy < ED_POLICY_FSM || opts->policy > ED_POLICY_SC))
    return fail(ED_E_INVALID_ARG, "unknown batching policy");
  if (opts && opts->staging != ED_STAGING_AUTO && opts->staging != ED_STAGING_OFF)
    return fail(ED_E_INVALID_ARG, "unknown staging mode");
  ed_plan_t *pl = new (std::nothrow) ed_plan_t();
  if (!pl) return fail(ED_E_OOM, "out of host memory");
  pl->types.assign(types, types + num_types);
  pl->staging = !(opts && opts->staging == ED_STAGING_OFF);
  pl->level_order = !(opts && opts->step_order == ED_ORDER_SCHEDULE);
  pl->hidden = types[0].hidden;
  pl->dtype = types[0].dtype;
  for (int t = 0; t < num_types; ++t) {
    const ed_op_type_t &ot = types[t];
    const std::string tag = "type " + std::to_string(t);
    if (ot.cell_kind < ED_CELL_TREELSTM_LEAF || ot.cell_kind > ED_CELL_MAX) { delete pl; return fail(ED_E_TYPE, tag + ": unknown cell kind"); }
    if (ot.hidden != pl->hidden || ot.dtype != pl->dtype) { delete pl; return fail(ED_E_TYPE, tag + ": hidden/dtype differ between types"); }
    if (ot.hidden <= 0) { delete pl; return fail(ED_E_TYPE, tag + ": hidden must be > 0"); }
    if (ot.dtype != ED_BF16 && ot.dtype != ED_FP32) { delete pl; return fail(ED_E_TYPE, tag + ": unknown dtype"); }
    if (ot.weight_set < 0 || ot.weight_set >= ed::kMaxWeightSets) { delete pl; return fail(ED_E_TYPE, tag + ": weight_set out of range"); }
    if (ot.num_slots < 0 || ot.num_slots > 2) { delete pl; return fail(ED_E_TYPE, tag + ": num_slots must be 0..2"); }
    if ((ot.cell_kind == ED_CELL_LINEAR_OUT || ot.cell_kind == ED_CELL_TAGGER) && (ot.out_dim <= 0 || ot.out_dim > 16)) { delete pl; return fail(ED_E_TYPE, tag + ": out_dim must be 1..16"); }
    if (ot.cell_kind == ED_CELL_MVRNN_INTERNAL && (ot.num_slots != 2 || ot.variadic || ot.has_ext)) { delete pl; return fail(ED_E_TYPE, tag + ": MV-RNN cells take exactly 2 fixed slots"); }
    if (ot.cell_kind == ED_CELL_MVRNN_INTERNAL && ot.hidden % 8 != 0) { delete pl; return fail(ED_E_TYPE, tag + ": MV-RNN needs hidden % 8 == 0"); }
    if (ot.cell_kind == ED_CELL_MVRNN_INTERNAL && ot.hidden > 2048) { delete pl; return fail(ED_E_UNSUPPORTED, tag + ": MV-RNN needs hidden <= 2048"); }
    if (ot.dtype == ED_BF16 && ot.hidden % 64 != 0) { delete pl; return fail(ED_E_TYPE, tag + ": bf16 path needs hidden % 64 == 0"); }
    if (!ed::cell_implemented(ot.cell_kind)) { delete pl; return fail(ED_E_UNSUPPORTED, tag + ": cell kind not implemented by this build"); }
  }
  ed_status_t st = validate_and_merge(pl, graphs, num_graphs);
  if (st != ED_OK) { delete pl; return st; }
  const double t1 = now_us();
  st = schedule(pl, fsm, opts ? opts->policy : ED_POLICY_FSM);
  if (st != ED_OK) { delete pl; return st; }
  const double t2 = now_us();
  if (layout == ED_LAYOUT_PQ) {
    ed::LayoutInput li{pl->V, &pl->gtype, &pl->in_off, &pl->in_idx, &pl->batch_type, &pl->batch_off, &pl->members,
                       &pl->types};
    try {
      pl->row_of_node = ed::plan_layout_pq(li);
    } catch (const std::exception &ex) {
      delete pl;
      return fail(ED_E_INVALID_ARG, std::string("PQ layout planner internal error: ") + ex.what());
    }
    if (pl->row_of_node.size() != static_cast<size_t>(pl->V)) { delete pl; return fail(ED_E_UNSUPPORTED, "PQ layout planner not available"); }
  } else {
    // ED_LAYOUT_SCHEDULE_ORDER: batches in schedule order; inside a batch, members ordered by the
    // latest batch producing one of their inputs (L-1: rows whose inputs are ready early share the
    // early tiles), then by the position of their earliest consumer (L-3: the rows one consumer tile
    // reads come from few producer tiles, so the consumer's early tiles start while the producer
    // step's later tiles still run), then by id.  Positions are fixed from the last batch backwards.
    pl->row_of_node.assign(pl->V, -1);
    std::vector<int32_t> bidx(pl->V, -1), rank(pl->V, 0);
    const int nbat = static_cast<int>(pl->batch_type.size());
    for (int b = 0; b < nbat; ++b)
      for (int k = pl->batch_off[b]; k < pl->batch_off[b + 1]; ++k) bidx[pl->members[k]] = b;
    static const int l3 = std::getenv("ED_LAYOUT_L3") ? std::atoi(std::getenv("ED_LAYOUT_L3")) : 1;
    // key = (latest producing batch + 1) * (V + 1) + (earliest consumer's global position, V if none);
    // members are ascending by id, so a stable LSD radix sort on the key yields (key, id) order
    std::vector<std::pair<uint64_t, int32_t>> key, tmp;
    const uint64_t V1 = static_cast<uint64_t>(pl->V) + 1;
    for (int b = nbat - 1; b >= 0; --b) {
      const int k0 = pl->batch_off[b], k1 = pl->batch_off[b + 1];
      key.clear();
      uint64_t kmax = 0;
      for (int k = k0; k < k1; ++k) {
        const int32_t v = pl->members[k];
        int32_t l = -1;
        for (int q = pl->in_off[v]; q < pl->in_off[v + 1]; ++q)
          if (pl->in_idx[q] >= 0) l = std::max(l, bidx[pl->in_idx[q]]);
        uint64_t ck = V1 - 1;  // no consumer: after every consumed member
        if (l3)
          for (int q = pl->coff[v]; q < pl->coff[v + 1]; ++q) {
            const int32_t w = pl->cons[q];
            ck = std::min(ck, static_cast<uint64_t>(pl->batch_off[bidx[w]]) + static_cast<uint64_t>(rank[w]));
          }
        const uint64_t kk = static_cast<uint64_t>(l + 1) * V1 + ck;
        kmax = std::max(kmax, kk);
        key.emplace_back(kk, v);
      }
      const size_t n = key.size();
      tmp.resize(n);
      if (n < 1024)  // small batches: a comparison sort on (key, id) is cheaper than the histograms
        std::sort(key.begin(), key.end());
      else
      for (int shift = 0; shift < 64 && (kmax >> shift) != 0; shift += 11) {
        std::vector<uint32_t> cnt(2049, 0);
        for (size_t i = 0; i < n; ++i) ++cnt[((key[i].first >> shift) & 2047u) + 1];
        for (int d = 0; d < 2048; ++d) cnt[d + 1] += cnt[d];
        for (size_t i = 0; i < n; ++i) tmp[cnt[(key[i].first >> shift) & 2047u]++] = key[i];
        key.swap(tmp);
      }
      for (size_t k = 0; k < n; ++k) rank[key[k].second] = static_cast<int32_t>(k);
    }
    int32_t r = 0;
    for (int b = 0; b < nbat; ++b) {
      const int k0 = pl->batch_off[b], k1 = pl->batch_off[b + 1];
      for (int k = k0; k < k1; ++k) pl->row_of_node[pl->members[k]] = r + rank[pl->members[k]];
      r += k1 - k0;
    }
  }
  const double t3 = now_us();
  st = lower(pl);
  if (st != ED_OK) { delete pl; return st; }
  pl->sched_us = t2 - t1;
  pl->layout_us = t3 - t2;
  pl->validate_us = t1 - t0;
  pl->plan_us = now_us() - t0;
  pl->lower_us = pl->plan_us - (t3 - t0);
  *out = pl;
  return ED_OK;
}

int64_t ed_plan_upload_bytes(const ed_plan_t *pl) { return pl ? static_cast<int64_t>(pl->blob.size()) : 0; }

ed_status_t ed_plan_info(const ed_plan_t *pl, ed_plan_info_t *o) {
  if (!pl || !o) return fail(ED_E_INVALID_ARG, "null argument");
  std::memset(o, 0, sizeof(*o));
  o->num_nodes = pl->V;
  o->num_instances = pl->ninst;
  o->num_batches = static_cast<int64_t>(pl->batch_type.size());
  o->num_steps = static_cast<int64_t>(pl->steps.size());
  o->lower_bound = pl->lower_bound;
  o->num_rows = pl->V + 1;
  o->hidden = pl->hidden;
  o->dtype = pl->dtype;
  o->workspace_bytes = static_cast<int64_t>(pl->ws_bytes);
  o->contig_operands = pl->contig;
  o->gather_operands = pl->gather;
  o->copy_bytes = pl->copy_bytes;
  o->copy_kernels = pl->copy_kernels;
  o->off_h = static_cast<int64_t>(pl->off_h);
  o->off_c = static_cast<int64_t>(pl->off_c);
  o->off_y = static_cast<int64_t>(pl->off_y);
  o->y_cols = pl->y_cols;
  o->off_x = pl->need_x ? static_cast<int64_t>(pl->off_x) : -1;
  o->off_u = pl->need_mv ? static_cast<int64_t>(pl->off_u) : -1;
  o->off_m = pl->need_mv ? static_cast<int64_t>(pl->off_m) : -1;
  o->off_ts = static_cast<int64_t>(pl->off_ts);
  o->plan_us = pl->plan_us;
  o->schedule_us = pl->sched_us;
  o->layout_us = pl->layout_us;
  o->validate_us = pl->validate_us;
  o->lower_us = pl->lower_us;
  o->staged_operands = pl->staged;
  o->staged_bytes = pl->staged_bytes;
  o->h_rows = pl->V + 1 + pl->op_rows;
  o->split_steps = 0;
  for (const auto &st : pl->steps) o->split_steps += (st.wsel & ed::kStepSplitK) ? 1 : 0;
  o->grid = pl->grid;
  return ED_OK;
}

ed_status_t ed_plan_get_schedule(const ed_plan_t *pl, int32_t *bt, int32_t *bo, int32_t *mem) {
  if (!pl || !bt || !bo || !mem) return fail(ED_E_INVALID_ARG, "null argument");
  std::copy(pl->batch_type.begin(), pl->batch_type.end(), bt);
  std::copy(pl->batch_off.begin(), pl->batch_off.end(), bo);
  std::copy(pl->members.begin(), pl->members.end(), mem);
  return ED_OK;
}

ed_status_t ed_plan_get_layout(const ed_plan_t *pl, int32_t *row) {
  if (!pl || !row) return fail(ED_E_INVALID_ARG, "null argument");
  std::copy(pl->row_of_node.begin(), pl->row_of_node.end(), row);
  return ED_OK;
}

ed_status_t ed_plan_get_slot_modes(const ed_plan_t *pl, int32_t *modes) {
  if (!pl || !modes) return fail(ED_E_INVALID_ARG, "null argument");
  std::copy(pl->slot_modes.begin(), pl->slot_modes.end(), modes);
  return ED_OK;
}

ed_status_t ed_plan_get_step_batches(const ed_plan_t *pl, int32_t *out) {
  if (!pl || !out) return fail(ED_E_INVALID_ARG, "null argument");
  std::copy(pl->step_batch.begin(), pl->step_batch.end(), out);
  return ED_OK;
}

void ed_plan_destroy(ed_plan_t *pl) {
  if (!pl) return;
  {
    WsRegistry &reg = ws_registry();
    std::lock_guard<std::mutex> lk(reg.mu);
    for (auto it = reg.owner.begin(); it != reg.owner.end();)
      it = (it->second.plan == pl) ? reg.owner.erase(it) : std::next(it);
  }
  delete pl;
}

int64_t ed_packed_bytes(int32_t cell_kind, int32_t hidden, int32_t out_dim, int32_t dtype, int32_t which) {
  return ed::packed_bytes(cell_kind, hidden, out_dim, dtype, which);
}

ed_status_t ed_pack_weights(int32_t cell_kind, int32_t hidden, int32_t out_dim, int32_t dtype, int32_t which,
                            const float *logical_dev, void *packed_dev, void *stream) {
  if (!logical_dev || !packed_dev) return fail(ED_E_INVALID_ARG, "null pointer");
  if (cell_kind < ED_CELL_TREELSTM_LEAF || cell_kind > ED_CELL_MAX) return fail(ED_E_TYPE, "unknown cell kind");
  int sms = 0, major = 0, minor = 0;
  int e = ed::device_check(&sms, &major, &minor);
  if (e) return fail(ED_E_CUDA, std::string("cuda: ") + cudaGetErrorString(static_cast<cudaError_t>(e)));
  if (major != 10 || minor != 0) return fail(ED_E_UNSUPPORTED, "device is not sm_100");
  e = ed::launch_pack(cell_kind, hidden, out_dim, dtype, which, logical_dev, packed_dev, stream);
  if (e) return fail(ED_E_CUDA, std::string("pack: ") + cudaGetErrorString(static_cast<cudaError_t>(e)));
  return ED_OK;
}

int32_t ed_execute_launch_count(const ed_plan_t *pl) { return pl ? 1 : 0; }  // one persistent kernel

ed_status_t ed_workspace_release(const void *ws) {
  if (!ws) return fail(ED_E_INVALID_ARG, "null workspace");
  WsRegistry &reg = ws_registry();
  std::lock_guard<std::mutex> lk(reg.mu);
  reg.owner.erase(ws);
  return ED_OK;
}

ed_status_t ed_execute(ed_plan_t *pl, const ed_weights_t *w, const ed_io_t *io, void *ws, size_t ws_bytes,
                       void *stream) {
  static const bool prof = std::getenv("ED_EXEC_TIMING") != nullptr;  // development: host phase times
  double tp[8] = {};
  if (prof) tp[0] = now_us();
  if (!pl || !w) return fail(ED_E_INVALID_ARG, "null argument");
  if (!ws || (reinterpret_cast<uintptr_t>(ws) & 1023) != 0) return fail(ED_E_WORKSPACE, "workspace null or not 1024-aligned");
  if (ws_bytes < pl->ws_bytes) return fail(ED_E_WORKSPACE, "workspace too small: need " + std::to_string(pl->ws_bytes));
  if (w->num_sets <= 0 || w->num_sets > ed::kMaxWeightSets || !w->sets) return fail(ED_E_INVALID_ARG, "bad weights");
  for (const auto &ot : pl->types)
    if (ot.weight_set >= w->num_sets) return fail(ED_E_INVALID_ARG, "weight set missing");
  if (!pl->bad_ext.empty()) return fail(ED_E_UNSUPPORTED, pl->bad_ext);
  for (const auto &ot : pl->types) {
    const ed_weight_set_t &s_ = w->sets[ot.weight_set];
    const std::string tag = "weight set " + std::to_string(ot.weight_set);
    if (ot.cell_kind == ED_CELL_MVRNN_INTERNAL && (!s_.mat || s_.emb_rows <= 0 || !s_.emb || !s_.W || !s_.b || !s_.W2))
      return fail(ED_E_INVALID_ARG, "MV-RNN weight set needs W, b, W2 (W_M), emb and mat with emb_rows > 0");
    if (!s_.W || !s_.b) return fail(ED_E_INVALID_ARG, tag + ": W and b must be non-null");
    if ((ot.cell_kind == ED_CELL_TAGGER || ot.cell_kind == ED_CELL_LATTICE_WORD) && (!s_.W2 || !s_.b2))
      return fail(ED_E_INVALID_ARG, tag + ": this cell needs W2 and b2");
  }
  for (int k = 0; k < ed::kMaxWeightSets; ++k) {  // every table id the plan reads is in range
    const bool used1 = pl->max_emb[k] >= 0, used2 = pl->max_emb2[k] >= 0;
    if (!used1 && !used2) continue;
    if (k >= w->num_sets) return fail(ED_E_INVALID_ARG, "weights: missing weight set " + std::to_string(k));
    const ed_weight_set_t &s_ = w->sets[k];
    if (used1 && (!s_.emb || pl->max_emb[k] >= s_.emb_rows))
      return fail(ED_E_INVALID_ARG, "weight set " + std::to_string(k) + ": token / external id " +
                                        std::to_string(pl->max_emb[k]) + " needs emb with more than that many rows (emb_rows " +
                                        std::to_string(s_.emb_rows) + ")");
    if (used2 && (!s_.emb2 || pl->max_emb2[k] >= s_.emb2_rows))
      return fail(ED_E_INVALID_ARG, "weight set " + std::to_string(k) + ": external char id " +
                                        std::to_string(pl->max_emb2[k]) + " needs emb2 with more than that many rows (emb2_rows " +
                                        std::to_string(s_.emb2_rows) + ")");
  }
  int sms = 0, major = 0, minor = 0;
  int e = ed::device_check(&sms, &major, &minor);
  if (e) return fail(ED_E_CUDA, std::string("cuda: ") + cudaGetErrorString(static_cast<cudaError_t>(e)));
  if (major != 10 || minor != 0) return fail(ED_E_UNSUPPORTED, "device is not sm_100 (sm_" + std::to_string(major * 10 + minor) + ")");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  uint8_t *base = static_cast<uint8_t *>(ws);
  if (prof) tp[1] = now_us();
  bool need_upload;
  uint64_t nonce = 0;
  uint32_t seq = 0;
  {
    WsRegistry &reg = ws_registry();
    std::lock_guard<std::mutex> lk(reg.mu);
    auto it = reg.owner.find(ws);
    need_upload = (it == reg.owner.end() || it->second.plan != pl);
    if (!need_upload) {
      nonce = it->second.nonce;
      seq = ++it->second.seq;
    } else {
      nonce = reg.next_nonce++;
    }
  }
  // the binding work runs on io->upload_stream when given (after this workspace's last launch),
  // and the launch stream waits for it
  cudaStream_t su = (io && io->upload_stream) ? static_cast<cudaStream_t>(io->upload_stream) : s;
  cudaEvent_t ws_done = nullptr, up_ev = nullptr;
  if (need_upload && su != s) {
    WsRegistry &reg = ws_registry();
    std::lock_guard<std::mutex> lk(reg.mu);
    auto it = reg.done.find(ws);
    if (it != reg.done.end()) ws_done = it->second;
    cudaEvent_t &ev = reg.up_ev[reg.up_next];
    reg.up_next = (reg.up_next + 1) % 16;
    if (!ev && cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess)
      return fail(ED_E_CUDA, "cudaEventCreate failed");
    up_ev = ev;
  }
  if (need_upload) {
    // bind: upload the static part with the binding nonce in its header, zero the readiness counters
    std::memcpy(pl->blob.data(), &nonce, sizeof(nonce));
    if (ws_done && cudaStreamWaitEvent(su, ws_done, 0) != cudaSuccess)
      return fail(ED_E_CUDA, "cudaStreamWaitEvent failed");
    cudaError_t ce = upload_async(base + pl->off_bar, pl->blob.data(), pl->blob.size(), su);
    if (prof) tp[2] = now_us();
    if (ce == cudaSuccess) ce = cudaMemsetAsync(base + pl->off_ready, 0, 4 * static_cast<size_t>(pl->V + 1), su);
    if (ce == cudaSuccess) {
      const size_t elt = pl->dtype == ED_BF16 ? 2 : 4;
      // zero row V and the staged rows (zero-state entries are never written by a producer)
      ce = cudaMemsetAsync(base + pl->off_h + elt * pl->V * pl->hidden, 0, elt * pl->hidden * (1 + pl->op_rows), su);
      if (ce == cudaSuccess) ce = cudaMemsetAsync(base + pl->off_c + 4 * pl->V * pl->hidden, 0, 4 * static_cast<size_t>(pl->hidden), su);
      if (ce == cudaSuccess && pl->need_x)
        ce = cudaMemsetAsync(base + pl->off_x + 4 * pl->V * pl->hidden, 0, 4 * static_cast<size_t>(pl->hidden), su);
      if (ce == cudaSuccess && pl->need_mv) {
        const size_t hh = static_cast<size_t>(pl->hidden);
        ce = cudaMemsetAsync(base + pl->off_u + elt * pl->V * 2 * hh, 0, elt * 2 * hh, su);
        if (ce == cudaSuccess) ce = cudaMemsetAsync(base + pl->off_m + elt * pl->V * hh * hh, 0, elt * hh * hh, su);
      }
    }
    if (ce != cudaSuccess) return fail(ED_E_CUDA, std::string("upload: ") + cudaGetErrorString(ce));
    WsRegistry &reg = ws_registry();
    std::lock_guard<std::mutex> lk(reg.mu);
    WsBinding &b = reg.owner[ws];
    b.plan = pl;
    b.nonce = nonce;
    b.seq = seq = 1;
  }
  if (prof) tp[3] = now_us();
  if (pl->grid == 0) {
    e = ed::persistent_grid(pl->dtype, pl->has_split, &pl->grid);
    if (e) return fail(ED_E_CUDA, std::string("occupancy: ") + cudaGetErrorString(static_cast<cudaError_t>(e)));
  }
  ed::KParams p;
  std::memset(&p, 0, sizeof(p));
  p.steps = reinterpret_cast<const ed::DevStep *>(base + pl->off_steps);
  p.idx = reinterpret_cast<const int32_t *>(base + pl->off_idx);
  p.root_rows = reinterpret_cast<const int32_t *>(base + pl->off_roots);
  p.H = base + pl->off_h;
  p.C = reinterpret_cast<float *>(base + pl->off_c);
  p.Y = reinterpret_cast<float *>(base + pl->off_y);
  p.X = pl->need_x ? reinterpret_cast<float *>(base + pl->off_x) : nullptr;
  p.U = pl->need_mv ? base + pl->off_u : nullptr;
  p.Mx = pl->need_mv ? base + pl->off_m : nullptr;
  p.hdr = reinterpret_cast<const unsigned long long *>(base + pl->off_bar);
  p.nonce = nonce;
  p.seq = seq;
  p.ext_root_off = pl->ext_root_off;
  p.num_ext_roots = pl->num_ext_roots;
  p.ts = reinterpret_cast<unsigned long long *>(base + pl->off_ts);
  p.ready = reinterpret_cast<int *>(base + pl->off_ready);
  p.target = reinterpret_cast<const int *>(base + pl->off_target);
  p.dst_off = p.idx + pl->dst_base;
  p.out_root = io ? io->out_root : nullptr;
  p.trace = io ? reinterpret_cast<unsigned long long *>(io->trace) : nullptr;
  p.num_steps = static_cast<int32_t>(pl->steps.size());
  p.hidden = pl->hidden;
  p.rows = static_cast<int32_t>(pl->V + 1);
  p.zero_row = static_cast<int32_t>(pl->V);
  p.ycols = static_cast<int32_t>(pl->y_cols);
  p.num_inst = pl->ninst;
  p.root_wset = pl->types[0].weight_set;
  for (int k = 0; k < w->num_sets; ++k) {
    const ed_weight_set_t &ws_ = w->sets[k];
    p.w[k] = ed::DevWeightSet{ws_.W, ws_.b, ws_.W2, ws_.b2, ws_.emb, ws_.emb2, ws_.mat, ws_.emb_rows, ws_.emb2_rows};
  }
  if (pl->dtype == ED_BF16) {
    const int64_t hh = pl->hidden;
    if (!encode_rows(&p.tm_h128, p.H, pl->V + 1 + pl->op_rows, hh, 128))
      return fail(ED_E_CUDA, "cuTensorMapEncodeTiled failed for the H buffer");
    if (pl->need_mv) {
      if (!encode_rows(&p.tm_u, p.U, pl->V + 1, 2 * hh, 128) || !encode_rows(&p.tm_mx, p.Mx, (pl->V + 1) * hh, hh, 64))
        return fail(ED_E_CUDA, "cuTensorMapEncodeTiled failed for the MV-RNN buffers");
      for (const auto &ot : pl->types) {
        if (ot.cell_kind != ED_CELL_MVRNN_INTERNAL) continue;
        const ed_weight_set_t &s_ = w->sets[ot.weight_set];
        if (!encode_rows(&p.tm_mat[ot.weight_set], s_.mat, static_cast<int64_t>(s_.emb_rows) * hh, hh, 64))
          return fail(ED_E_CUDA, "cuTensorMapEncodeTiled failed for a word-matrix table");
      }
    }
  }
  p.has_split = pl->has_split ? 1 : 0;
  if (up_ev) {  // the launch waits for the side-stream binding work
    if (cudaEventRecord(up_ev, su) != cudaSuccess || cudaStreamWaitEvent(s, up_ev, 0) != cudaSuccess)
      return fail(ED_E_CUDA, "ordering the upload stream before the launch failed");
  }
  if (prof) tp[4] = now_us();
  e = ed::launch_persistent(p, pl->dtype, pl->grid, pl->has_split, stream);
  if (e == 0 && io && io->upload_stream) {  // for the next side-stream upload into this workspace
    WsRegistry &reg = ws_registry();
    std::lock_guard<std::mutex> lk(reg.mu);
    cudaEvent_t &ev = reg.done[ws];
    if (!ev && cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) ev = nullptr;
    if (ev) cudaEventRecord(ev, s);
  }
  if (prof) {
    tp[5] = now_us();
    std::fprintf(stderr, "ed_execute us: checks %.1f bind+upload %.1f memsets %.1f params %.1f launch %.1f (blob %zu B)\n",
                 tp[1] - tp[0], tp[2] > 0 ? tp[2] - tp[1] : 0.0, tp[2] > 0 ? tp[3] - tp[2] : 0.0, tp[4] - tp[3],
                 tp[5] - tp[4], pl->blob.size());
  }
  if (e) return fail(ED_E_CUDA, std::string("launch: ") + cudaGetErrorString(static_cast<cudaError_t>(e)));
  return ED_OK;
}

}  // extern "C"
