/*
 * ed_batch.h — C ABI of the B200-native ED-Batch hot path (libedbatch.so).
 *
 * What it computes (arXiv 2302.03851, PAPER.md):
 *   ed_plan     Alg. 1 "FSM-based Dynamic Batching" over the disjoint union of
 *               per-instance dataflow graphs, with the E_sort state encoding and a
 *               given FSM transition table pi(S); then a memory layout of the
 *               node outputs (§3: results and sources of each batch contiguous and
 *               aligned where possible); then lowering to a device step table.
 *   ed_execute  runs the whole batch schedule as ONE persistent sm_100a kernel: per batch,
 *               gather (or block-read) operand rows, the cell's dense contraction (tcgen05/TMEM
 *               for bf16, FFMA for fp32), fused gate epilogue, contiguous result store; grid-wide
 *               barrier between batches (removing the per-batch launch overhead of P:40).
 *
 * Conventions for every call:
 *   - Return value: ED_OK (0) or a negative ed_status_t; on failure a thread-local message is
 *     available from ed_last_error() until the next failing call on the same thread.
 *   - Host arrays passed in are BORROWED for the duration of the call only.
 *   - Device pointers are caller-owned (PyTorch tensors); the library never allocates device
 *     memory (no cudaMalloc) and never synchronises the host with the device inside ed_execute.
 *   - Streams are cudaStream_t passed as void* (0 = legacy default stream).
 */
#ifndef ED_BATCH_H
#define ED_BATCH_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t ed_status_t;

#define ED_OK               0
#define ED_E_INVALID_ARG   -1  /* null pointer, bad size, bad CSR offsets, bad ext id        */
#define ED_E_CYCLE         -2  /* an instance graph is not acyclic (Alg. 1 needs a DAG)       */
#define ED_E_DANGLING      -3  /* node input / root refers to a node id outside the instance  */
#define ED_E_DUP_ID        -4  /* reserved: CSR ids are implicit, so duplicates cannot occur  */
#define ED_E_TYPE          -5  /* op type index out of range or unsupported cell/dtype mix    */
#define ED_E_ARITY         -6  /* number of inputs does not match the op type's slots         */
#define ED_E_FSM           -7  /* malformed FSM table (bad key, action not in its key)        */
#define ED_E_CUDA          -8  /* a CUDA runtime call failed                                  */
#define ED_E_UNSUPPORTED   -9  /* device is not sm_100 or the plan needs an unbuilt variant   */
#define ED_E_WORKSPACE    -10  /* workspace pointer null/misaligned or smaller than required  */
#define ED_E_OOM          -11  /* host allocation failed                                      */

/* Slot value meaning "zero state" (h_{-1} = c_{-1} = 0), read from a dedicated zero row. */
#define ED_ZERO_INPUT INT32_MIN

/* Cell kinds (equations: DESIGN.md §3 / SURVEY App. A; the paper only cites them). */
#define ED_CELL_TREELSTM_LEAF      1  /* Table 4 P:364.  x = emb[ext]; [i;o;u] = W x + b          */
#define ED_CELL_TREELSTM_INTERNAL  2  /* Table 4 P:363.  slots (l, r); [i;f_l;f_r;o;u] = U[h_l;h_r] */
#define ED_CELL_LINEAR_OUT         3  /* output op O (Fig. 1): y = W h + b, fp32 logits     */
#define ED_CELL_TREEGRU_LEAF       4  /* Table 4                                            */
#define ED_CELL_TREEGRU_INTERNAL   5  /* Table 4                                            */
#define ED_CELL_TREEFC_INTERNAL    6  /* h = tanh(W[h_l;h_r] + b); slots may be external words   */
#define ED_CELL_LSTM               7  /* BiLSTM F/B cell: x = emb[ext], slot = h_prev     */
#define ED_CELL_TAGGER             8  /* y = W2 tanh(W1[h_f;h_b] + b1) + b2                       */
#define ED_CELL_MVRNN_INTERNAL     9  /* MV-RNN (Table 4)                            */
#define ED_CELL_LATTICE_CHAR      10  /* LatticeLSTM char cell (Fig. 7), variadic    */
#define ED_CELL_LATTICE_WORD      11  /* LatticeLSTM word cell                                     */
#define ED_CELL_LATTICEGRU_CHAR   12  /* LatticeGRU char cell (A-27): GRU over      */
                                      /* [x_e; h_{e-1}], max-pooled with the words ending at e      */
#define ED_CELL_LATTICEGRU_WORD   13  /* LatticeGRU word cell: GRU over [x_w; h_b] (slot: C_b)      */
#define ED_CELL_MAX               13

#define ED_FP32 0
#define ED_BF16 1

#define ED_ENC_SORT 0   /* E_sort: frontier types by descending count, ties ascending id */
#define ED_ENC_BASE 1   /* E_base: ascending set of frontier types                                 */
#define ED_ENC_MAX  2   /* E_max: (E_base, the most frequent frontier type); as an entry key:
                           the ascending type set followed by that type (key_len = |set| + 1;
                           count ties to the lowest type id)                                        */

#define ED_FALLBACK_KEY0 0  /* table miss or action not ready: take key[0] (reading A-3) */

#define ED_LAYOUT_SCHEDULE_ORDER 0  /* rows in schedule order: results contiguous, sources gathered */
#define ED_LAYOUT_PQ             1
#define ED_STAGING_AUTO          0
#define ED_STAGING_OFF           1  /* PQ-tree plan (§3.2, Alg. 2-6) over the node-output rows      */

/* One op type ("each operation is given a type"). */
typedef struct {
  int32_t cell_kind;   /* ED_CELL_*                                                         */
  int32_t num_slots;   /* fixed input slots (variadic cells: the fixed prefix)              */
  int32_t variadic;    /* 1: node inputs after the fixed slots are a variable-length list   */
  int32_t has_ext;     /* 1: the op reads emb[ext[v]] of its weight set                     */
  int32_t weight_set;  /* index into ed_weights_t.sets                                      */
  int32_t hidden;      /* h; every type of one plan must share it                          */
  int32_t out_dim;     /* logits width for ED_CELL_LINEAR_OUT / ED_CELL_TAGGER, else 0      */
  int32_t dtype;       /* ED_BF16 | ED_FP32; every type of one plan must share it          */
} ed_op_type_t;

/* One instance graph in CSR form (node ids are 0..num_nodes-1, implicit).
 *   type[v]          op type index
 *   in_off[v..v+1]   range of in_idx holding v's inputs in slot order (in_off[0] == 0)
 *   in_idx[k] >= 0   local node id;  == ED_ZERO_INPUT: zero state;  other < 0: external
 *                    input id (-1 - id) read from the type's embedding table (word leaves)
 *   ext[v]           token id for has_ext types, else ignored (may be NULL if no type has ext)
 *   root             local node id whose h is the instance output, or (-1 - id) for an
 *                    instance with no ops whose output is the external row itself          */
typedef struct {
  int32_t num_nodes;
  const int32_t *type;
  const int32_t *in_off;
  const int32_t *in_idx;
  const int32_t *ext;
  int32_t root;
} ed_graph_t;

/* FSM transition table pi (Fig. 2; P:140 constant-time lookup): key = E(G) as a
 * list of type ids, action = the type to batch next. */
typedef struct {
  int32_t key_len;
  const int32_t *key;
  int32_t action;
} ed_fsm_entry_t;

typedef struct {
  int32_t encoder;       /* ED_ENC_SORT | ED_ENC_BASE | ED_ENC_MAX */
  int32_t num_entries;
  const ed_fsm_entry_t *entries;
  int32_t fallback;      /* ED_FALLBACK_KEY0 */
} ed_fsm_t;

typedef struct {
  int32_t layout;        /* ED_LAYOUT_SCHEDULE_ORDER | ED_LAYOUT_PQ */
  int32_t staging;       /* ED_STAGING_AUTO (0): bf16 plans stage gathered cell operands of large
                            batches (the producer's epilogue also stores its h row into a
                            contiguous operand block of the consuming batch, read by TMA);
                            ED_STAGING_OFF (1): every non-contiguous operand is gathered row by
                            row.  Results are bitwise identical. */
  int32_t policy;        /* batching policy (PAPER P:107, P:436 comparators; Fig. 8):
                            ED_POLICY_FSM (0): Alg. 1 with the FSM table (fsm), the default;
                            ED_POLICY_DEPTH: TF-Fold depth-based: one batch per (topological
                              depth, type), ascending depth then type id (fsm ignored);
                            ED_POLICY_AGENDA: DyNet agenda-based Alg. 1: the ready type with the
                              smallest mean depth over all nodes of the type, ties to the lower id;
                            ED_POLICY_SC: sufficient-condition heuristic Alg. 1: argmax of Eq. 1's
                              second term |Frontier_a(G_t)| / |Frontier(G^a_t)| (A-1),
                              ties to the larger ready count, then the lower id.
                            Depth of an op = 1 + max depth of its node inputs (raw inputs: 0). */
  int32_t step_order;    /* order in which the kernel walks the batches (their member sets are the
                            schedule's either way): ED_ORDER_LEVEL (0): stable by dependency level
                            (1 + the highest level among the batches producing a member's inputs),
                            so independent chains (BiLSTM directions, separate lattices) interleave
                            and overlap in the dataflow kernel; ED_ORDER_SCHEDULE (1): the schedule
                            order.  ed_plan_get_step_batches reports the device order. */
  int32_t reserved[4];   /* must be 0 */
} ed_plan_opts_t;
#define ED_POLICY_FSM    0
#define ED_POLICY_DEPTH  1
#define ED_POLICY_AGENDA 2
#define ED_POLICY_SC     3
#define ED_ORDER_LEVEL    0
#define ED_ORDER_SCHEDULE 1

typedef struct ed_plan_s ed_plan_t;  /* opaque plan handle */

typedef struct {
  int64_t num_nodes;          /* V (all instances)                                        */
  int64_t num_instances;
  int64_t num_batches;        /* length of the schedule                                   */
  int64_t num_steps;          /* device steps (a two-contraction cell = 2 steps per batch) */
  int64_t lower_bound;        /* sum_t Depth(G_t) (App. B.3)                   */
  int64_t num_rows;           /* V + 1 (row V is the all-zero row)                        */
  int64_t hidden;
  int64_t dtype;
  int64_t workspace_bytes;    /* minimum size of the ed_execute workspace                 */
  int64_t contig_operands;    /* (batch, fixed slot) operands read as one block           */
  int64_t gather_operands;    /* (batch, fixed slot) operands read by row index           */
  int64_t copy_bytes;         /* gather+scatter bytes a copy-based executor would move    */
  int64_t copy_kernels;       /* gather+scatter kernels a copy-based executor would launch */
  int64_t off_h;              /* workspace byte offsets of the row buffers:               */
  int64_t off_c;              /*   H [num_rows x hidden] (dtype), C [num_rows x hidden] f32 */
  int64_t off_y;              /*   Y [num_rows x y_cols] f32 (logits of output ops)       */
  int64_t y_cols;
  int64_t off_x;              /*   X [num_rows x hidden] f32 (lattice link gates)         */
  int64_t off_ts;             /*   u64 %globaltimer stamp after each device step (num_steps+1) */
  int64_t off_u;              /*   U [num_rows x 2 hidden] (dtype): MV-RNN [B a; A b], or -1  */
  int64_t off_m;              /*   Mx [num_rows x hidden x hidden] (dtype): MV-RNN node       */
                              /*   matrices, each stored TRANSPOSED (row k = column k of P), or -1 */
  double plan_us;             /* host time spent in ed_plan                               */
  double schedule_us;
  double layout_us;
  int64_t staged_operands;    /* bf16: gathered (batch, slot) operands staged into contiguous   */
                              /*   blocks by their producers' epilogues (read as TMA boxes)     */
  int64_t staged_bytes;       /* bytes of those extra producer stores per execute               */
  int64_t h_rows;             /* rows of the H buffer: num_rows + staged operand rows           */
  double validate_us;         /* host time of validation + merge (part of plan_us)              */
  double lower_us;            /* host time of lowering (step table, index arrays, workspace map) */
  int64_t split_steps;        /* bf16: device steps run split-K over a CTA pair:   */
                              /*   each CTA of a 2-CTA cluster multiplies one K half; the pair     */
                              /*   exchanges partial sums over distributed shared memory           */
  int64_t grid;               /* CTAs of the persistent launch (0 until the first ed_execute)    */
} ed_plan_info_t;

/* Per weight set, device pointers.  Matrices must have been packed by ed_pack_weights.
 *   W     packed main matrix of the cell (logical [G*h, K] rows = gate-stacked outputs)
 *   b     fp32 bias [G*h] (logical order)
 *   W2,b2 second matrix (TAGGER: [C, h]; LATTICE_WORD: link gate [h, 2h]; MVRNN: W_M [h, 2h])
 *   emb   embedding table [emb_rows, h] (dtype of the plan); emb2 second table (lattice chars)
 *   mat   MV-RNN word matrices, packed by ed_pack_weights(ED_CELL_MVRNN_INTERNAL, h, emb_rows,
 *         dtype, 2, ...) from the logical [emb_rows, h, h] table: each matrix transposed.
 *   MV-RNN (Socher et al. 2012; Table 4): W = [h, 2h] and b = [h] of
 *         p = tanh(W [B a; A b] + b); W2 = W_M [h, 2h] of P = W_M [A; B]; emb = word vectors. */
typedef struct {
  const void *W;
  const float *b;
  const void *W2;
  const float *b2;
  const void *emb;
  const void *emb2;
  const void *mat;
  int32_t emb_rows;
  int32_t emb2_rows;
} ed_weight_set_t;

typedef struct {
  int32_t num_sets;
  const ed_weight_set_t *sets;
} ed_weights_t;

typedef struct {
  void *out_root;   /* [num_instances x hidden] in the plan dtype: root h of each instance, in
                       instance order (may be NULL) */
  uint64_t *trace;  /* optional device buffer [num_steps x 64] of %globaltimer stamps taken by
                       CTA 0 at fixed phases of each batch (profiling aid; NULL = off) */
  void *upload_stream;  /* optional cudaStream_t for the binding work of an execute that binds (the
                       static part's H2D and the zeroing): it is ordered after the previous launch
                       on this workspace, and the launch stream waits for it.  With two workspaces
                       used in turn, the next minibatch's upload overlaps the running kernel.
                       NULL: everything on the launch stream. */
} ed_io_t;

/* Build a plan (host only; no CUDA call).  Validates the graphs (errors above), merges them
 * (instance-major global ids), runs Alg. 1 with the table, plans the layout, lowers it. */
ed_status_t ed_plan(const ed_graph_t *graphs, int32_t num_graphs, const ed_op_type_t *types,
                    int32_t num_types, const ed_fsm_t *fsm, const ed_plan_opts_t *opts,
                    ed_plan_t **out);

ed_status_t ed_plan_info(const ed_plan_t *plan, ed_plan_info_t *out);

/* Schedule of the plan (Alg. 1 output): batch_type[num_batches], batch_off[num_batches+1],
 * members[num_nodes] = global node ids, each batch in position (= ascending row) order. */
ed_status_t ed_plan_get_schedule(const ed_plan_t *plan, int32_t *batch_type, int32_t *batch_off,
                                 int32_t *members);

/* row_of_node[num_nodes]: row of each global node's output record in the H/C/Y buffers. */
ed_status_t ed_plan_get_layout(const ed_plan_t *plan, int32_t *row_of_node);

/* Per (batch, fixed slot) flag: 1 = contiguous block read, 0 = gathered. [num_batches * 2] */
ed_status_t ed_plan_get_slot_modes(const ed_plan_t *plan, int32_t *modes);

/* batch_of_step[num_steps]: the schedule batch (index into ed_plan_get_schedule) each device step
 * executes, in the order the kernel walks them (opts.step_order); a two-contraction cell's batch
 * has two consecutive device steps.  Also the meaning of the trace / step-stamp indices. */
ed_status_t ed_plan_get_step_batches(const ed_plan_t *plan, int32_t *batch_of_step);

void ed_plan_destroy(ed_plan_t *plan);

/* Bytes of the packed form of a logical matrix.  which = 0: main W; 1: W2; 2 (MV-RNN only): the
 * word-matrix table, logical [out_dim, h, h] (out_dim = number of words). */
int64_t ed_packed_bytes(int32_t cell_kind, int32_t hidden, int32_t out_dim, int32_t dtype, int32_t which);

/* Pack a logical fp32 matrix (device, row-major [rows, cols] as in DESIGN.md §5) into the
 * device layout the kernels read: bf16 gate-interleaved, K-major, 128B-swizzled UMMA canonical
 * tiles; fp32 transposed for FFMA.  Asynchronous on stream. */
ed_status_t ed_pack_weights(int32_t cell_kind, int32_t hidden, int32_t out_dim, int32_t dtype, int32_t which,
                            const float *logical_dev, void *packed_dev, void *stream);

/* Execute the plan: one persistent cooperative kernel on `stream`, nothing else (no memsets).
 * The first execute of a plan on a workspace binds them: it uploads the plan's static part (step
 * table, index arrays, readiness targets, a binding nonce in the workspace header; async H2D) and
 * zeroes the readiness counters, the zero row and the staged rows.  Later executes reuse the
 * binding (readiness counters are monotonic across launches).  The workspace contents must
 * persist between executes; before freeing or reusing the memory for anything else call
 * ed_workspace_release (a launch on a workspace whose header no longer holds the nonce traps).
 * Results: node records in the workspace row buffers (offsets in ed_plan_info_t) and, when
 * io->out_root is non-null, the instance outputs out_root[num_instances x hidden] (plan dtype),
 * written by the epilogues that produce the root rows. */
ed_status_t ed_execute(ed_plan_t *plan, const ed_weights_t *weights, const ed_io_t *io, void *workspace,
                       size_t workspace_bytes, void *stream);

/* Bytes of the plan's static part (step table, index arrays) that the first ed_execute on a
 * workspace uploads host->device (through a reused pinned staging buffer). */
int64_t ed_plan_upload_bytes(const ed_plan_t *plan);

/* Number of kernels ed_execute launches (for launch accounting). */
int32_t ed_execute_launch_count(const ed_plan_t *plan);

/* Forget the plan binding of a workspace (call before freeing or reusing its memory; a later
 * execute on the same address binds again).  Host-only, no device work; ED_E_INVALID_ARG on null. */
ed_status_t ed_workspace_release(const void *workspace);

/* ---------------------------------------------------------------------------------------------
 * Learning the FSM (PAPER §2.3 "Using RL to Learn the FSM"; §5.3): tabular
 * N-step Q-learning over the instance graphs, one instance per episode (episodes cycle over the
 * graphs).  State = E(G_t) (ED_ENC_SORT, ED_ENC_BASE or ED_ENC_MAX), action = the next batch's type (all
 * ready nodes of it, Alg. 1), reward Eq. 1 r = -1 + alpha * |Frontier_a(G_t)| / |Frontier(G^a_t)|
 * (the ratio read as in DESIGN.md A-1).  After each episode, for t = 0..T-1 in order:
 *   Q(S_t,a_t) += lr * (sum_{i<N, t+i<T} r_{t+i} + [t+N<T] max_b Q(S_{t+N},b) - Q(S_t,a_t))
 * (b over the types present in S_{t+N}; unseen pairs count 0; no discount).  Actions are
 * epsilon-greedy over the ready types: one SplitMix64 draw x, u = (x >> 11) * 2^-53; u < eps takes
 * ready[y % #ready] for a second draw y (ready types ascending), else argmax Q (ties: lowest id);
 * eps = max(eps_floor, eps0 * eps_decay^(episode / eps_every)).  Every check_every episodes the
 * greedy table is evaluated with Alg. 1 (A-3 fallback for unseen states) on all instances and
 * training stops when the batch total reaches the App. B.3 lower bound (sum over instances).
 * The result is an FSM table for ed_plan plus the Q values: pi(S) = argmax_a Q(S, a) over the
 * actions tried in S, taken from the best greedy table evaluated (the checkpoints and
 * the final Q; fewest batches, earliest on ties).
 * Host only; deterministic for a given seed; no CUDA call. ------------------------------------ */
typedef struct {
  int32_t encoder;       /* ED_ENC_SORT | ED_ENC_BASE | ED_ENC_MAX                               */
  int32_t n_steps;       /* N >= 1 (bootstrapping horizon)                                        */
  int32_t max_episodes;  /* paper: 1000                                                   */
  int32_t check_every;   /* paper: 50                                                     */
  int32_t eps_every;     /* episodes per epsilon decay step                                       */
  int32_t episode_graph; /* ED_RL_EPISODE_INSTANCE: one instance graph per episode (cycling);
                            ED_RL_EPISODE_MERGED: every episode runs Alg. 1 over the merged minibatch
                            (the dataflow graph ed_plan schedules); checkpoints and the
                            lower bound are then those of the merged graph                          */
  double alpha;          /* Eq. 1 coefficient, >= 0                                               */
  double lr;             /* learning rate in (0, 1]                                               */
  double eps0, eps_decay, eps_floor;
  uint64_t seed;         /* SplitMix64 seed                                                       */
} ed_rl_config_t;        /* defaults (A-26): SORT, 4, 1000, 50, 10, INSTANCE, .5, .1, .5, .95, .02 */
#define ED_RL_EPISODE_INSTANCE 0
#define ED_RL_EPISODE_MERGED   1

typedef struct ed_fsm_learned_s ed_fsm_learned_t;  /* opaque; owned by the caller */

typedef struct {
  int64_t episodes;         /* episodes run (early stop included)                               */
  int64_t table_entries;    /* states with a learned action                                     */
  int64_t q_entries;        /* (state, action) pairs with a Q value                             */
  int64_t checkpoints;      /* greedy evaluations run                                           */
  int64_t final_batches;    /* greedy batch total of the returned table over the instances      */
  int64_t lower_bound;      /* sum of the instances' App. B.3 lower bounds                      */
  double learn_us;          /* host time                                                        */
} ed_fsm_learned_info_t;

/* Learn an FSM table.  Graphs/types as for ed_plan (validated the same way; errors likewise);
 * ED_E_INVALID_ARG for a bad config. */
ed_status_t ed_fsm_learn(const ed_graph_t *graphs, int32_t num_graphs, const ed_op_type_t *types,
                         int32_t num_types, const ed_rl_config_t *cfg, ed_fsm_learned_t **out);
ed_status_t ed_fsm_learned_info(const ed_fsm_learned_t *fl, ed_fsm_learned_info_t *out);
/* The learned table as an ed_fsm_t for ed_plan (encoder of the config, fallback key[0]).  The
 * entries and keys are owned by fl and valid until ed_fsm_learned_destroy. */
ed_status_t ed_fsm_learned_table(const ed_fsm_learned_t *fl, ed_fsm_t *out);
/* Q entry k in (state key lexicographic, action ascending) order: key[*key_len] (capacity
 * num_types + 1: an E_max key is the type set followed by its most frequent type), action and value. */
ed_status_t ed_fsm_learned_q(const ed_fsm_learned_t *fl, int64_t k, int32_t *key, int32_t *key_len,
                             int32_t *action, double *q);
/* Checkpoint c: episode count and greedy batch total at that checkpoint. */
ed_status_t ed_fsm_learned_checkpoint(const ed_fsm_learned_t *fl, int64_t c, int64_t *episode,
                                      int64_t *batches);
void ed_fsm_learned_destroy(ed_fsm_learned_t *fl);

/* Version string and build arch, e.g. "ed_batch 0.1 sm_100a". */
const char *ed_version(void);

const char *ed_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* ED_BATCH_H */
