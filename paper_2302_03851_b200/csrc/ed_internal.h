// Internal definitions shared by the host planner (ed_batch.cpp) and the device code
// (ed_kernels.cu).  Not part of the public ABI (include/ed_batch.h is).
#pragma once
#include <cuda.h>
#include <stdint.h>

#include "ed_batch.h"

namespace ed {

constexpr int kMaxWeightSets = 8;

// Device-only step kinds: the second contraction of a two-GEMM cell runs as its own step.
constexpr int kCellLatticeLink = 101;  // l = s(W_l [x_e; c^w] + b_l) of LatticeLSTM word cells -> X
constexpr int kCellTaggerOut = 102;    // y = W2 t + b2 of the BiLSTM tagger (t in the node's H row) -> Y
// MV-RNN (Socher et al. 2012; Table 4) runs as three device steps over the same rows:
//   ED_CELL_MVRNN_INTERNAL  u = [B a; A b]                         (matvecs, HBM-bound)    -> U
//   kCellMvP                p = tanh(W u + b)                      (tensor cores, K = 2h)  -> H
//   kCellMvMat              P^T = [A^T | B^T] W_M^T  (= (W_M [A;B])^T, tensor cores)       -> Mx
// Node matrices are stored transposed (Mx row block of a node = M^T, row-major h x h).
constexpr int kCellMvP = 103;
constexpr int kCellMvMat = 104;
constexpr int kMaxSlotsDev = 2;
constexpr int kStepSplitK = 2;    // DevStep::wsel flag   // fixed slots the device reads (all cells have <= 2)

// One batch of the schedule as the persistent kernel sees it (SoA-friendly 64 B record).
// Slot j of member i (position i = ascending result row):
//   mode[j] == 1 (CONTIG): entry = arg[j] + i             (one contiguous aligned block)
//   mode[j] == 0 (GATHER): entry = idx[arg[j] + i]
//   mode[j] == 2 (STAGED): entry = idx[arg[j] + i] as for GATHER, and the A operand of the slot is
//                          read from H rows idx[arg[j] + m] + i: a block the producers' epilogues
//                          fill with copies of their h rows (bf16 tensor-core cells only)
// An entry >= 0 is a row of the H/C/X buffers (the zero row for ED_ZERO_INPUT); an entry < 0 is
// an external id (-1 - id) read from the weight set's embedding table.
struct DevStep {
  int32_t cell;       // ED_CELL_*
  int32_t m;          // batch size
  int32_t out_row0;   // results occupy rows out_row0 .. out_row0 + m - 1 (always contiguous)
  int32_t wset;       // weight set
  int32_t mode[kMaxSlotsDev];
  int32_t arg[kMaxSlotsDev];
  int32_t ext_off;    // idx offset of the per-member ext token ids, -1 if none
  int32_t var_off;    // idx offset of m+1 absolute offsets of variadic input lists, -1 if none
  int32_t units;      // UMMA path: hidden units per column tile (multiple of 16)
  int32_t n_col_tiles;// UMMA path: hidden / units
  int32_t gates;      // G: gate blocks of the main contraction
  int32_t nslots;     // fixed slots present
  int32_t wsel;       // bit 0 -- 0: weight set W/b, 1: second matrix W2/b2; bit 1 (kStepSplitK):
                      // split-K over the CTA pair of a cluster (rank r multiplies K half r; the
                      // pair exchanges the partial sums of each other's 8-unit half over DSMEM)
  int32_t self_need;  // readiness a row of this step's own output block must reach before the step
                      // may read it (= what earlier device steps of the same batch publish)
};
static_assert(sizeof(DevStep) == 64, "DevStep must be 64 bytes");

struct DevWeightSet {
  const void *W;
  const float *b;
  const void *W2;
  const float *b2;
  const void *emb;
  const void *emb2;
  const void *mat;
  int32_t emb_rows;
  int32_t emb2_rows;
};

// Kernel parameters (passed as __grid_constant__ so the TMA descriptors below are addressable).
struct alignas(64) KParams {
  CUtensorMap tm_h128;                   // H rows, box {64 cols, 128 rows}: contiguous blocks
  CUtensorMap tm_u;                      // U rows (2h cols), box {64, 128}
  CUtensorMap tm_mx;                     // node matrices Mx as [(rows * h) x h], box {64, 64}
  CUtensorMap tm_mat[kMaxWeightSets];    // word-matrix tables as [(words * h) x h], box {64, 64}
  const DevStep *steps;
  const int32_t *idx;
  const int32_t *root_rows;   // per instance: row (>= 0) or external id (-1 - id)
  void *H;                    // [rows x hidden] bf16 or fp32
  float *C;                   // [rows x hidden]
  float *Y;                   // [rows x ycols]
  float *X;                   // [rows x hidden] (lattice link gates) or null
  void *U;                    // [rows x 2 hidden] (MV-RNN matvec results [B a; A b]) or null
  void *Mx;                   // [rows x hidden x hidden] (MV-RNN node matrices, transposed) or null
  const unsigned long long *hdr;  // workspace header: the binding nonce written when the plan was uploaded
  unsigned long long nonce;   // expected header value (a stale or replaced workspace traps)
  unsigned long long *ts;     // [num_steps + 1] (max of %globaltimer: monotonic, never zeroed)
  void *out_root;             // [num_inst x hidden] or null
  unsigned long long *trace;  // [num_steps x 64] phase stamps of CTA 0, or null
  const int32_t *dst_off;     // [rows + 1] copies of each result row (CSR into idx): entry >= 0 a staged
                              // H row, entry < 0 the instance output out_root[-1 - entry]
  int *ready;                 // [rows] units published per row, monotonic over launches: after launch
                              // k a row holds k * target (mod 2^32); zeroed only when the workspace is bound
  const int *target;          // [rows] units a row holds when final (sum of step_contrib)
  int32_t num_steps;
  int32_t hidden;
  int32_t rows;
  int32_t zero_row;
  int32_t ycols;
  int32_t num_inst;
  int32_t root_wset;
  uint32_t seq;               // launches of this plan on this workspace binding, 1, 2, ...
  int32_t ext_root_off;       // idx offset of (instance, external id) pairs of instances whose
  int32_t num_ext_roots;      // output is an input lookup (no op produces it)
  int32_t has_split;          // some step is split-K over a CTA pair: launched with clusters of 2
  DevWeightSet w[kMaxWeightSets];
};

// Gates of the main contraction per cell kind (0: not a single-GEMM cell).
inline int cell_gates(int cell) {
  switch (cell) {
    case ED_CELL_TREELSTM_LEAF: return 3;
    case ED_CELL_TREELSTM_INTERNAL: return 5;
    case ED_CELL_TREEGRU_LEAF: return 2;
    case ED_CELL_TREEGRU_INTERNAL: return 5;
    case ED_CELL_TREEFC_INTERNAL: return 1;
    case ED_CELL_LSTM: return 4;
    case ED_CELL_LATTICE_CHAR: return 4;
    case ED_CELL_LATTICE_WORD: return 3;
    case ED_CELL_LATTICEGRU_CHAR:
    case ED_CELL_LATTICEGRU_WORD: return 4;  // [r; z; n_x; n_h] (n_x: x part only, n_h: h part only)
    case ED_CELL_TAGGER: return 1;
    case ED_CELL_MVRNN_INTERNAL: return 1;
    case kCellLatticeLink: return 1;
    case kCellMvP: return 1;
    case kCellMvMat: return 1;
    default: return 0;
  }
}

// Hidden units per column tile on the bf16 tensor-core path (N tile = gates * units <= 256); the
// last column tile of a row holds the remaining h % units units.  Fixed per cell kind so that host
// tiling and the device epilogue templates agree.
#ifndef ED_MAX_TILE_N
#define ED_MAX_TILE_N 256  // widest MMA N tile (B stage = N x 128 B)
#endif
inline int cell_units_max(int cell);
inline int cell_units(int cell) {
  const int u = cell_units_max(cell), g = cell_gates(cell);
  if (u <= 0 || g <= 0 || g * u <= ED_MAX_TILE_N) return u;
  return (ED_MAX_TILE_N / g) / 16 * 16;
}
inline int cell_units_max(int cell) {
  switch (cell) {
    case ED_CELL_TREELSTM_LEAF: return 80;      // N = 240
    case ED_CELL_TREELSTM_INTERNAL: return 48;  // N = 240
    case ED_CELL_TREEGRU_LEAF: return 128;      // N = 256
    case ED_CELL_TREEGRU_INTERNAL: return 48;   // N = 240
    case ED_CELL_TREEFC_INTERNAL: return 192;   // N = 192 (measured faster than 256)
    case ED_CELL_LSTM: return 64;               // N = 256
    case ED_CELL_LATTICE_CHAR: return 64;       // N = 256
    case ED_CELL_LATTICE_WORD: return 80;       // N = 240
    case ED_CELL_LATTICEGRU_CHAR:
    case ED_CELL_LATTICEGRU_WORD: return 64;    // N = 256
    case kCellLatticeLink: return 192;          // N = 192 (measured faster than 256)
    case ED_CELL_TAGGER: return 256;            // N = 256
    case kCellMvP: return 256;                  // N = 256
    case kCellMvMat: return 256;                // N = 256 (columns of P^T)
    default: return 0;
  }
}

// Cell kinds the device code implements in this build.
inline bool cell_implemented(int cell) {
  switch (cell) {
    case ED_CELL_TREELSTM_LEAF:
    case ED_CELL_TREELSTM_INTERNAL:
    case ED_CELL_LINEAR_OUT:
    case ED_CELL_TREEGRU_LEAF:
    case ED_CELL_TREEGRU_INTERNAL:
    case ED_CELL_TREEFC_INTERNAL:
    case ED_CELL_LSTM:
    case ED_CELL_TAGGER:
    case ED_CELL_LATTICE_CHAR:
    case ED_CELL_LATTICE_WORD:
    case ED_CELL_LATTICEGRU_CHAR:
    case ED_CELL_LATTICEGRU_WORD:
    case ED_CELL_MVRNN_INTERNAL: return true;
    default: return false;
  }
}

// Cells whose 16-unit tiles may run split-K over a CTA pair (the device instantiates the split
// epilogue for these only).
inline bool cell_splittable(int cell) {
  switch (cell) {
    case ED_CELL_TREELSTM_INTERNAL:
    case ED_CELL_TREEGRU_INTERNAL: return true;
    default: return false;
  }
}

// K segments (each of width hidden) of the main contraction.
inline int cell_segments(int cell) {
  switch (cell) {
    case ED_CELL_TREELSTM_LEAF:
    case ED_CELL_TREEGRU_LEAF:
    case ED_CELL_LINEAR_OUT: return 1;
    default: return 2;
  }
}

// Readiness units a device step publishes per row of its output block when it completes: h for
// row-vector results; h * h (elements) for the MV-RNN matrix product.
// Output-linear ops (logits in Y, A-7) are sinks: nothing waits for them, so they publish nothing.
inline int step_contrib(int cell, int h) {
  if (cell == ED_CELL_LINEAR_OUT || cell == kCellTaggerOut) return 0;
  return cell == kCellMvMat ? h * h : h;
}

// Launch entry points implemented in ed_kernels.cu (return cudaError_t as int).
int launch_persistent(const KParams &p, int dtype, int grid, bool cluster2, void *stream);
int launch_pack(int cell, int hidden, int out_dim, int dtype, int which, const float *src, void *dst,
                void *stream);
int64_t packed_bytes(int cell, int hidden, int out_dim, int dtype, int which);
int device_check(int *sm_count, int *major, int *minor);
int persistent_grid(int dtype, bool cluster2, int *grid);

}  // namespace ed
