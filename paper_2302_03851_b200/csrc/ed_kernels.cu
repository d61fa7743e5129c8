// ed_kernels.cu — device side of the ED-Batch hot path for sm_100a (B200).
//
// One persistent cooperative kernel walks the whole FSM batch schedule (PAPER Alg. 1,
// P:75-87): for every batch ("step") it reads operand rows (gathered by index, or one contiguous
// block where the layout plan made them adjacent), runs the cell's dense contraction,
// applies the fused gate epilogue and stores the results as one contiguous row block.  Dependent
// steps are ordered by per-row readiness counters (release / acquire), not by kernel launches or
// grid barriers: this replaces the per-batch kernel launches of the paper's DyNet executor.
//
//   bf16 path (ed_persistent_bf16): every cell's contraction on the 5th-gen tensor cores —
//     warps 0-3  epilogue (setmaxnreg 232): tcgen05.ld TMEM -> registers, gates in fp32, vector stores
//     warp  4    MMA issuer: tcgen05.mma.cta_group::1.kind::f16 (M=128), elect.sync issue
//     warp  5    weight loader: cp.async.bulk of pre-swizzled weight tiles (complete_tx)
//     warps 6-11 operand loaders: TMA 128-row box for CONTIG / staged operands, 16 B cp.async row
//                gathers otherwise (192 threads), into 128B-swizzled A tiles
//     4-stage smem ring (mbarrier full/empty), 2 TMEM accumulators (2 x 256 columns).
//     The output linear O runs as an N = 16 tensor-core tile; the tagger output and the MV-RNN
//     matvecs are SIMT phases of all warps.
//   fp32 path (ed_persistent_f32): FFMA SIMT for every cell (1e-4 parity path; single-pass TF32
//     and approximate transcendentals cannot meet 1e-4, A-20).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <cstdlib>

#include "ed_internal.h"

namespace ed {

// ------------------------------------------------------------------------------------------------
// constants of the bf16 tensor-core engine
// ------------------------------------------------------------------------------------------------
constexpr int kThreads = 256;        // fp32 SIMT kernel
#ifndef ED_LOADER_WARPS
#define ED_LOADER_WARPS 6
#endif
constexpr int kLoaderThreads = ED_LOADER_WARPS * 32;  // warps 6.. (operand gathers)
constexpr int kThreadsTC = 192 + kLoaderThreads;      // bf16 tensor-core kernel: 4 epilogue, MMA, B, loaders
#ifndef ED_STAGES
#define ED_STAGES 4
#endif
constexpr int kStages = ED_STAGES;
constexpr int kTileM = 128;
constexpr int kChunkK = 64;                  // bf16 elements per 128 B swizzle row
constexpr int kAStage = kTileM * 128;        // 16 KB
constexpr int kBStage = ED_MAX_TILE_N * 128;  // 32 KB (N tile <= 256)
constexpr int kStageBytes = kAStage + kBStage;
constexpr int kRowTab = kTileM * 2 * 8;      // row pointers per tile (2 segments)
constexpr int kBiasBytes = 5 * 512 * 4;           // G * h fp32 (G * h <= 2560)
constexpr int kWoutBytes = 12 * 1024;             // output-linear weights [C][h] fp32 (else read from L2)
#ifndef ED_SMEM_SLACK
#define ED_SMEM_SLACK 1024  // alignment slack of the dynamic shared memory base
#endif
constexpr int kSmemBytes = ED_SMEM_SLACK + kStages * kStageBytes + 2 * kRowTab + kBiasBytes + kWoutBytes + 256;
constexpr int kEpiThreads = 128;
// setmaxnreg budgets (multiples of 8): 128 x kEpiRegs + 256 x kProdRegs <= 64K registers per SM
#ifndef ED_EPI_REGS
#define ED_EPI_REGS 232
#endif
#ifndef ED_PROD_REGS
#define ED_PROD_REGS 136
#endif
constexpr int kEpiRegs = ED_EPI_REGS;
constexpr int kProdRegs = ED_PROD_REGS;
static_assert(kEpiThreads * kEpiRegs + (kThreadsTC - kEpiThreads) * kProdRegs <= 65536, "register budget");
static_assert(kStages <= ED_LOADER_WARPS, "one owning loader warp per ring stage");
static_assert(kThreadsTC % 128 == 0, "setmaxnreg acts on whole warpgroups: 4 + 2 + loader warps = 4k warps");


// ------------------------------------------------------------------------------------------------
// PTX helpers
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cnt(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
#ifndef ED_TEST_WAIT
#define ED_TEST_WAIT 0
#endif
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar), ok = 0, spins = 0;
  do {
    if (++spins > (1u << 30)) __trap();  // watchdog: a lost arrival must not hang the GPU
#if ED_TEST_WAIT  // non-blocking probe (no suspend / resume of the waiting thread)
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(addr), "r"(parity)
        : "memory");
    continue;
#endif
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(addr), "r"(parity)
        : "memory");
  } while (!ok);
}
// Warp-wide wait: one lane polls the barrier, the warp then reconverges (fewer try_wait probes
// competing for the barrier / shared-memory pipe than 32 polling lanes).
#ifndef ED_LANE0_POLL
#define ED_LANE0_POLL 0
#endif
__device__ __forceinline__ void mbar_wait_warp(uint64_t *bar, uint32_t parity) {
#if ED_LANE0_POLL
  if ((threadIdx.x & 31) == 0) mbar_wait(bar, parity);
  __syncwarp();
#else
  mbar_wait(bar, parity);
#endif
}
// Wait with a back-off between probes (for waiters off the K-loop's critical path: fewer probes
// competing with the ring's barrier traffic).
__device__ __forceinline__ void mbar_wait_sleep(uint64_t *bar, uint32_t parity, uint32_t ns) {
  uint32_t addr = smem_u32(bar), ok = 0, spins = 0;
  for (;;) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(addr), "r"(parity)
        : "memory");
    if (ok) break;
    if (++spins > (1u << 28)) __trap();
    __nanosleep(ns);
  }
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// Warp-converged forms (one elected lane issues; operands warp-uniform)
__device__ __forceinline__ void mbar_arrive_tx_elect(uint64_t *bar, uint32_t bytes) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n\t}" ::"r"(smem_u32(bar)), "r"(bytes)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s_elect(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n\t}" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// TMA: one box {64 cols, box rows} of a 2-D bf16 tensor at (col, row) -> smem, complete_tx on bar
__device__ __forceinline__ void tma_row_box(void *dst, const CUtensorMap *m, int col, int row, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(m), "r"(col), "r"(row), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_row_box_elect(void *dst, const CUtensorMap *m, int col, int row, uint64_t *bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e cp.async.bulk.tensor.2d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n\t}" ::"r"(
          smem_u32(dst)),
      "l"(m), "r"(col), "r"(row), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
// Row-table read as an explicit shared-memory load: a generic LD of a shared address is ordered
// behind the thread's in-flight cp.async copies, which serialised one L2 round trip per K chunk.
__device__ __forceinline__ const void *lds_ptr(const void *const *p) {
  unsigned long long v;
  asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(smem_u32(p)));
  return reinterpret_cast<const void *>(v);
}
// 256-bit global stores (sm_100): one full 32 B sector per thread
__device__ __forceinline__ void st_v8_b32(void *a, uint4 lo, uint4 hi) {
  asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(a), "r"(lo.x), "r"(lo.y), "r"(lo.z),
               "r"(lo.w), "r"(hi.x), "r"(hi.y), "r"(hi.z), "r"(hi.w)
               : "memory");
}
__device__ __forceinline__ void st_v8_f32(float *a, const float *v) {
  asm volatile("st.global.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(a), "f"(v[0]), "f"(v[1]), "f"(v[2]),
               "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
               : "memory");
}
// 256-bit L2 (.cg) loads: one full 32 B sector per thread
__device__ __forceinline__ void ldcg_v8(const void *a, float4 &lo, float4 &hi) {
  asm volatile("ld.global.cg.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=f"(lo.x), "=f"(lo.y), "=f"(lo.z), "=f"(lo.w), "=f"(hi.x), "=f"(hi.y), "=f"(hi.z), "=f"(hi.w)
               : "l"(a));
}
__device__ __forceinline__ void ldcg_v8(const void *a, uint4 &lo, uint4 &hi) {
  asm volatile("ld.global.cg.v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(lo.x), "=r"(lo.y), "=r"(lo.z), "=r"(lo.w), "=r"(hi.x), "=r"(hi.y), "=r"(hi.z), "=r"(hi.w)
               : "l"(a));
}
__device__ __forceinline__ float4 lds_f4(const float *p) {
  float4 v;
  asm("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(smem_u32(p)));
  return v;
}
__device__ __forceinline__ void sts_ptr(const void **p, const void *v) {
  asm volatile("st.shared.u64 [%0], %1;" ::"r"(smem_u32(p)), "l"(reinterpret_cast<unsigned long long>(v)) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
// The mbarrier receives one arrival once every cp.async this thread issued so far has landed (the
// barrier's expected count includes it: .noinc).
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t *bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Warp-converged forms: every lane walks the issue loop (operands stay warp-uniform, no per-MMA
// single-lane R2UR loop) and elect.sync picks the issuing lane.
__device__ __forceinline__ void tc_mma_elect(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tc_commit_elect(uint64_t *bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}
// 32 lanes x 32 bit, 16 consecutive columns per thread
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float *v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, "
      "[%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
#pragma unroll
  for (int k = 0; k < 16; ++k) v[k] = __uint_as_float(r[k]);
}
// 32 lanes x 32 bit, 8 consecutive columns per thread
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float *v) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
#pragma unroll
  for (int k = 0; k < 8; ++k) v[k] = __uint_as_float(r[k]);
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// ---- CTA-pair (cluster of 2) exchange for split-K steps ----
// shared::cluster address of the same shared-memory object in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_u32(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// arrive on an mbarrier of another CTA of the cluster, ordering this thread's earlier accesses
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t *bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar), ok = 0, spins = 0;
  do {
    if (++spins > (1u << 30)) __trap();
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(addr), "r"(parity)
        : "memory");
  } while (!ok);
}
// 16 B into another CTA's shared memory; the bytes complete_tx on that CTA's mbarrier
__device__ __forceinline__ void st_async_v4(uint32_t cluster_addr, float a, float b, float c, float d,
                                            uint32_t cluster_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
                   cluster_addr),
               "f"(a), "f"(b), "f"(c), "f"(d), "r"(cluster_bar)
               : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void st_v4_b32(void *a, uint4 v) {
  asm volatile("st.global.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

// UMMA shared-memory descriptor: K-major, 128B swizzle, 8-row atoms 1024 B apart (SBO), version 1.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return static_cast<uint64_t>((saddr & 0x3FFFF) >> 4) | (static_cast<uint64_t>(1) << 16) |
         (static_cast<uint64_t>(1024 >> 4) << 32) | (static_cast<uint64_t>(1) << 46) |
         (static_cast<uint64_t>(2) << 61);
}
// Instruction descriptor kind::f16: D f32, A/B bf16, both K-major, M = 128, N = n.
__device__ __forceinline__ uint32_t idesc_bf16(int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(n >> 3) << 17) |
         (static_cast<uint32_t>(kTileM >> 4) << 24);
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// ---- dataflow readiness (replaces per-batch grid barriers) ----
// ready[row] counts units written to the row by finished device steps; target[row] = the sum of
// step_contrib over the device steps that write it (h per row-vector result, h*h for a matrix).
// A consumer acquires ready[row] - base >= target[row] before reading the row, base = (seq - 1) *
// target[row] (mod 2^32: the counters are never reset between launches, so no memset precedes a
// launch); a producer publishes with a release-add after its stores.  Rows are only produced by
// earlier device steps and every warp walks the steps in order, so waiting cannot deadlock.
__device__ __forceinline__ int ld_acquire_s32(const int *a) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
  return v;
}
#ifndef ED_WATCHDOG_PRINTF
#define ED_WATCHDOG_PRINTF 0
#endif
#ifndef ED_TMA_ONE_ARRIVE
#define ED_TMA_ONE_ARRIVE 0  // measured neutral
#endif
#ifndef ED_TMA_ROTATE
#define ED_TMA_ROTATE 1  // TMA box of a stage issued by loader warp (stage mod 6): cfg3 149.5 -> 146.4 us
#endif
#ifndef ED_EPI_WAIT_SLEEP
#define ED_EPI_WAIT_SLEEP 0
#endif
#ifndef ED_POLL_NS
#define ED_POLL_NS 32  // back-off between readiness polls
#endif
// A step that reads its own rows (the second contraction of a two-GEMM cell: link gate, tagger
// output, MV-RNN p) needs only what the earlier steps of its batch publish: st.self_need.
__device__ __forceinline__ int ready_since_launch(const KParams &p, int e, int tgt) {
  return static_cast<int>(static_cast<uint32_t>(ld_acquire_s32(p.ready + e)) - (p.seq - 1u) * static_cast<uint32_t>(tgt));
}
// Watchdog: report the stuck dependency, then abort the launch.  Out of line, so the printf
// argument marshalling does not cost registers in every polling loop.
__device__ __noinline__ void watchdog_abort(int cell, int out_row0, int row, int ready, int need) {
  printf("ed_batch watchdog: block %d thread %d cell %d out_row0 %d row %d ready %d need %d\n", blockIdx.x,
         threadIdx.x, cell, out_row0, row, ready, need);
  __trap();
}
__device__ __forceinline__ void wait_row(const KParams &p, int e, const DevStep &st) {
  if (e < 0 || e >= p.rows) return;  // external rows are static
  const int tgt = __ldg(p.target + e);
  int need = tgt;
  if (e >= st.out_row0 && e < st.out_row0 + st.m) need = st.self_need;
  if (need <= 0) return;
  unsigned spins = 0;
  while (ready_since_launch(p, e, tgt) < need) {
    if (++spins > (1u << 26)) {  // watchdog: a lost publication must not hang the GPU
#if ED_WATCHDOG_PRINTF  // diagnostic build: report the stuck dependency (the printf costs registers)
      printf("ed_batch watchdog: block %d thread %d cell %d out_row0 %d row %d ready %d need %d\n", blockIdx.x,
             threadIdx.x, st.cell, st.out_row0, e, ready_since_launch(p, e, tgt), need);
#endif
      __trap();
    }
#if ED_POLL_NS > 0
    __nanosleep(ED_POLL_NS);
#endif
  }
}
// Non-blocking check of a row (same rule as wait_row).
__device__ __forceinline__ bool row_ready(const KParams &p, int e, const DevStep &st) {
  if (e < 0 || e >= p.rows) return true;
  const int tgt = __ldg(p.target + e);
  int need = tgt;
  if (e >= st.out_row0 && e < st.out_row0 + st.m) need = st.self_need;
  return need <= 0 || ready_since_launch(p, e, tgt) >= need;
}
__device__ __forceinline__ void publish_row(const KParams &p, int row, int units) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p.ready + row), "r"(units) : "memory");
}
// Row copies listed in dst_off: a staged operand row of H (d >= 0) or the instance output
// out_root[-1 - d] (written here by the producer's epilogue, no final gather pass); null when the
// caller passed no out_root.
template <typename T>
__device__ __forceinline__ T *copy_row(const KParams &p, int d) {
  if (d >= 0) return static_cast<T *>(p.H) + static_cast<size_t>(d) * p.hidden;
  return p.out_root ? static_cast<T *>(p.out_root) + static_cast<size_t>(-1 - d) * p.hidden : nullptr;
}
// Kernel prologue: the workspace must still hold the binding this launch was planned for (a freed
// and reallocated workspace has lost its step table and readiness counters: fail loudly), and
// instance outputs that are input lookups (no op produces them) are copied by CTA 0.
template <typename T>
__device__ void prologue_checks(const KParams &p) {
  if (threadIdx.x == 0 && *p.hdr != p.nonce) {
    printf("ed_batch: workspace binding lost (header %llx, expected %llx): call ed_workspace_release "
           "before freeing a workspace\n", *p.hdr, p.nonce);
    __trap();
  }
  if (blockIdx.x != 0 || p.num_ext_roots == 0 || p.out_root == nullptr) return;
  const int h = p.hidden;
  for (int q = threadIdx.x; q < p.num_ext_roots * h; q += blockDim.x) {
    const int k = q / h, j = q % h;
    const int inst = __ldg(p.idx + p.ext_root_off + 2 * k), id = __ldg(p.idx + p.ext_root_off + 2 * k + 1);
    const T *tab = static_cast<const T *>(p.w[p.root_wset].emb);
    static_cast<T *>(p.out_root)[static_cast<size_t>(inst) * h + j] = tab[static_cast<size_t>(id) * h + j];
  }
}
__device__ __forceinline__ void stamp_step(const KParams &p, int s) {
  atomicMax(p.ts + s + 1, globaltimer());
}

// optional phase trace of CTA 0 (profiling aid)
// phase stamps of the CTA that runs item 0 of each step (profiling aid; off unless io.trace is set)
#ifdef ED_NO_TRACE
#define ED_TRACE(p, s, k, first) do { } while (0)
#else
#define ED_TRACE(p, s, k, first) \
  do { if ((p).trace && (first)) (p).trace[(s) * 64 + (k)] = globaltimer(); } while (0)
#endif

// ------------------------------------------------------------------------------------------------
// cell math — one hidden unit, fp32
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ int cell_segments_dev(int cell) {
  return (cell == ED_CELL_TREELSTM_LEAF || cell == ED_CELL_TREEGRU_LEAF || cell == ED_CELL_LINEAR_OUT ||
          cell == kCellTaggerOut) ? 1 : 2;
}

__device__ __forceinline__ float sigm(float x) { return 1.0f / (1.0f + expf(-x)); }
// bf16 path: MUFU tanh.approx (rel. err ~2^-11, below the bf16 rounding of h, 2^-9)
__device__ __forceinline__ float tanh_fast(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float sigm_fast(float x) { return fmaf(0.5f, tanh_fast(0.5f * x), 0.5f); }
// activations by storage type: fp32 path accurate (1e-4 parity), bf16 path MUFU approximations
template <typename T> __device__ __forceinline__ float act_sig(float x) { return sigm_fast(x); }
template <> __device__ __forceinline__ float act_sig<float>(float x) { return sigm(x); }
template <typename T> __device__ __forceinline__ float act_tanh(float x) { return tanh_fast(x); }
template <> __device__ __forceinline__ float act_tanh<float>(float x) { return tanhf(x); }
template <typename T> __device__ __forceinline__ float act_exp(float x) { return __expf(x); }
template <> __device__ __forceinline__ float act_exp<float>(float x) { return expf(x); }

// Slot j (0 or 1) of a step: selects instead of st.mode[j] / st.arg[j], so the step record stays in
// registers (a runtime index would put it in local memory, and with 224 KB of shared memory per
// CTA the L1 left for local memory is small: local loads go to L2).
__device__ __forceinline__ int slot_mode(const DevStep &st, int j) { return j == 0 ? st.mode[0] : st.mode[1]; }
__device__ __forceinline__ int slot_arg(const DevStep &st, int j) { return j == 0 ? st.arg[0] : st.arg[1]; }
__device__ __forceinline__ int slot_entry(const DevStep &st, const int32_t *idx, int j, int i) {
  const int mode = slot_mode(st, j), arg = slot_arg(st, j);
  return mode == 1 ? arg + i : __ldg(idx + arg + i);
}

template <typename T>
__device__ __forceinline__ float to_f(T v);
template <>
__device__ __forceinline__ float to_f<float>(float v) { return v; }
template <>
__device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }
template <typename T>
__device__ __forceinline__ T from_f(float v);
template <>
__device__ __forceinline__ float from_f<float>(float v) { return v; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

__device__ __forceinline__ const void *step_W(const KParams &p, const DevStep &st) {
  return (st.wsel & 1) ? p.w[st.wset].W2 : p.w[st.wset].W;
}
__device__ __forceinline__ const float *step_b(const KParams &p, const DevStep &st) {
  return (st.wsel & 1) ? p.w[st.wset].b2 : p.w[st.wset].b;
}
__device__ __forceinline__ bool step_split(const DevStep &st) { return (st.wsel & kStepSplitK) != 0; }

// Pointer to the h-vector an operand entry refers to (row of H, or an external embedding row).
template <typename T>
__device__ __forceinline__ const T *entry_row(const KParams &p, const DevWeightSet &w, int e, bool second) {
  if (e >= 0) return static_cast<const T *>(p.H) + static_cast<size_t>(e) * p.hidden;
  const int id = -1 - e;
  const T *tab = static_cast<const T *>(second ? w.emb2 : w.emb);
  return tab + static_cast<size_t>(id) * p.hidden;
}

// K segment s (width hidden) of member i's A operand.
template <typename T>
__device__ __forceinline__ const T *segment_row(const KParams &p, const DevStep &st, int s, int i) {
  const DevWeightSet &w = p.w[st.wset];
  const int cell = st.cell;
  const bool ext_first = (cell == ED_CELL_TREELSTM_LEAF || cell == ED_CELL_TREEGRU_LEAF ||
                          cell == ED_CELL_LSTM || cell == ED_CELL_LATTICE_CHAR || cell == ED_CELL_LATTICE_WORD ||
                          cell == ED_CELL_LATTICEGRU_CHAR || cell == ED_CELL_LATTICEGRU_WORD);
  if (ext_first) {
    if (s == 0) {
      const int tok = __ldg(p.idx + st.ext_off + i);
      return static_cast<const T *>(w.emb) + static_cast<size_t>(tok) * p.hidden;
    }
    return entry_row<T>(p, w, slot_entry(st, p.idx, 0, i), false);
  }
  // MV-RNN p step: K segment s of u = [B a; A b] in the node's own U row
  if (cell == kCellMvP) return static_cast<const T *>(p.U) + (static_cast<size_t>(st.out_row0 + i) * 2 + s) * p.hidden;
  // lattice link gate: x_e of the word's end char comes from the char table (emb2)
  return entry_row<T>(p, w, slot_entry(st, p.idx, s, i), cell == kCellLatticeLink && s == 0);
}

__device__ __forceinline__ bool ext_first_cell(int cell) {
  return cell == ED_CELL_TREELSTM_LEAF || cell == ED_CELL_TREEGRU_LEAF || cell == ED_CELL_LSTM ||
         cell == ED_CELL_LATTICE_CHAR || cell == ED_CELL_LATTICE_WORD || cell == ED_CELL_LATTICEGRU_CHAR ||
         cell == ED_CELL_LATTICEGRU_WORD;
}
// Operand entry of K segment s for member i: >= 0 row of H; < 0 embedding row (-1 - id).
__device__ __forceinline__ int segment_entry(const KParams &p, const DevStep &st, int s, int i) {
  if (st.cell == kCellMvP) return st.out_row0 + i;  // own U row (published by the matvec step)
  if (ext_first_cell(st.cell)) {
    if (s == 0) return -1 - __ldg(p.idx + st.ext_off + i);
    return slot_entry(st, p.idx, 0, i);
  }
  return slot_entry(st, p.idx, s, i);
}
// Whether K segment s is one contiguous block of H rows (layout plan made it adjacent + aligned).
__device__ __forceinline__ bool segment_contig(const KParams &p, const DevStep &st, int s, int *base) {
  if (st.cell == kCellMvP) {  // the node's own U rows: always one block
    *base = st.out_row0;
    return true;
  }
  int slot = s;
  if (ext_first_cell(st.cell)) {
    if (s == 0) return false;
    slot = 0;
  }
  const int mode = slot_mode(st, slot), arg = slot_arg(st, slot);
  if (mode == 2) {  // staged block (rows written by the producers' epilogues)
    *base = __ldg(p.idx + arg + st.m);
    return true;
  }
  *base = arg;
  return mode == 1;
}

__device__ __forceinline__ float c_of(const KParams &p, int e, int j) {
  return e >= 0 ? __ldcg(p.C + static_cast<size_t>(e) * p.hidden + j) : 0.0f;
}

// Scalar epilogue for one (member i, unit j) given the gate pre-activations z[] (bias included).
template <typename T>
__device__ __forceinline__ void cell_epilogue(const KParams &p, const DevStep &st, int i, int j, const float *z) {
  const int h = p.hidden;
  const size_t orow = static_cast<size_t>(st.out_row0 + i);
  T *H = static_cast<T *>(p.H);
  float c = 0.f, hv = 0.f;
  bool has_c = true;
  switch (st.cell) {
    case ED_CELL_TREELSTM_LEAF:  // [i;o;u]
      c = act_sig<T>(z[0]) * act_tanh<T>(z[2]);
      hv = act_sig<T>(z[1]) * act_tanh<T>(c);
      break;
    case ED_CELL_TREELSTM_INTERNAL: {  // [i;f_l;f_r;o;u]
      const int el = slot_entry(st, p.idx, 0, i), er = slot_entry(st, p.idx, 1, i);
      c = act_sig<T>(z[0]) * act_tanh<T>(z[4]) + act_sig<T>(z[1]) * c_of(p, el, j) + act_sig<T>(z[2]) * c_of(p, er, j);
      hv = act_sig<T>(z[3]) * act_tanh<T>(c);
      break;
    }
    case ED_CELL_TREEGRU_LEAF:  // [z;n]
      hv = (1.f - act_sig<T>(z[0])) * act_tanh<T>(z[1]);
      has_c = false;
      break;
    case ED_CELL_TREEGRU_INTERNAL: {  // [z;r_l;r_r;a_l;a_r]
      const int el = slot_entry(st, p.idx, 0, i), er = slot_entry(st, p.idx, 1, i);
      const DevWeightSet &w = p.w[st.wset];
      const float hl = to_f<T>(entry_row<T>(p, w, el, false)[j]);
      const float hr = to_f<T>(entry_row<T>(p, w, er, false)[j]);
      const float n = act_tanh<T>(act_sig<T>(z[1]) * z[3] + act_sig<T>(z[2]) * z[4]);
      const float zz = act_sig<T>(z[0]);
      hv = (1.f - zz) * n + zz * (hl + hr);
      has_c = false;
      break;
    }
    case ED_CELL_TREEFC_INTERNAL:
    case kCellMvP:  // MV-RNN p = tanh(W [B a; A b] + b)
      hv = act_tanh<T>(z[0]);
      has_c = false;
      break;
    case ED_CELL_LSTM: {  // [i;f;g;o]
      const int ep = slot_entry(st, p.idx, 0, i);
      c = act_sig<T>(z[1]) * c_of(p, ep, j) + act_sig<T>(z[0]) * act_tanh<T>(z[2]);
      hv = act_sig<T>(z[3]) * act_tanh<T>(c);
      break;
    }
    case ED_CELL_LATTICE_WORD: {  // [i;f;g]: c^w = s(f) c_b + s(i) tanh(g); h row <- c^w (link operand)
      const int eb = slot_entry(st, p.idx, 0, i);
      c = act_sig<T>(z[1]) * c_of(p, eb, j) + act_sig<T>(z[0]) * act_tanh<T>(z[2]);
      hv = c;
      break;
    }
    case ED_CELL_LATTICEGRU_CHAR:
    case ED_CELL_LATTICEGRU_WORD: {  // GRU [r; z; n_x; n_h] (A-27), char: max-pool with word states
      const DevWeightSet &w = p.w[st.wset];
      const int ep = slot_entry(st, p.idx, 0, i);
      const float hp = to_f<T>(entry_row<T>(p, w, ep, false)[j]);
      const float rr = act_sig<T>(z[0]), zz = act_sig<T>(z[1]);
      const float n = act_tanh<T>(z[2] + rr * z[3]);
      hv = (1.f - zz) * n + zz * hp;
      if (st.cell == ED_CELL_LATTICEGRU_CHAR) {
        const int beg = __ldg(p.idx + st.var_off + i), end = __ldg(p.idx + st.var_off + i + 1);
        for (int k = beg; k < end; ++k)
          hv = fmaxf(hv, to_f<T>(__ldcg(static_cast<const T *>(p.H) + static_cast<size_t>(__ldg(p.idx + k)) * h + j)));
      }
      has_c = false;
      break;
    }
    case kCellLatticeLink:  // l = s(W_l [x_e; c^w] + b_l) -> X
      p.X[orow * h + j] = act_sig<T>(z[0]);
      return;
    case ED_CELL_TAGGER:  // t = tanh(W1 [h_f; h_b] + b1) -> h row (read by the tagger output step)
      hv = act_tanh<T>(z[0]);
      has_c = false;
      break;
    case ED_CELL_LATTICE_CHAR: {  // [i;f;o;g]; variadic words: softmax over {s(i)} U {l_w}
      const int ep = slot_entry(st, p.idx, 0, i);
      const int beg = __ldg(p.idx + st.var_off + i), end = __ldg(p.idx + st.var_off + i + 1);
      const float si = act_sig<T>(z[0]), tg = act_tanh<T>(z[3]);
      if (beg == end) {
        c = act_sig<T>(z[1]) * c_of(p, ep, j) + si * tg;
      } else {
        const float ei = act_exp<T>(si);
        float den = ei, num = ei * tg;
        for (int k = beg; k < end; ++k) {
          const int wr = __ldg(p.idx + k);
          const float el = act_exp<T>(__ldcg(p.X + static_cast<size_t>(wr) * h + j));
          den += el;
          num += el * __ldcg(p.C + static_cast<size_t>(wr) * h + j);
        }
        c = num / den;
      }
      hv = act_sig<T>(z[2]) * act_tanh<T>(c);
      break;
    }
    default:
      return;
  }
  H[orow * h + j] = from_f<T>(hv);
  if (has_c) p.C[orow * h + j] = c;
  for (int d = __ldg(p.dst_off + orow); d < __ldg(p.dst_off + orow + 1); ++d) {
    T *dst = copy_row<T>(p, __ldg(p.idx + d));
    if (dst) dst[j] = from_f<T>(hv);
  }
}

// ------------------------------------------------------------------------------------------------
// SIMT engine (fp32 path for every cell; bf16 path for the cells without a tensor-core variant)
// Weights: Wt[k][n] (transposed logical [G*h, K]), element type T.
// ------------------------------------------------------------------------------------------------
template <typename T>
__device__ void simt_gemm_step(const KParams &p, const DevStep &st) {
  const int h = p.hidden, G = st.gates, NS = cell_segments_dev(st.cell);
  const T *Wt = static_cast<const T *>(step_W(p, st));
  const float *bias = step_b(p, st);
  const int lane = threadIdx.x & 31;
  const int nub = (h + 31) / 32;
  const long tasks = static_cast<long>(st.m) * nub;
  const long gw = (static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const long nw = (static_cast<long>(gridDim.x) * blockDim.x) >> 5;
  const int ldw = G * h;
  for (long task = gw; task < tasks; task += nw) {
    const int i = static_cast<int>(task / nub);
    const int j = static_cast<int>(task % nub) * 32 + lane;
    // inputs of member i: slot rows (A operand, c rows) and variadic words
    for (int sl = 0; sl < st.nslots; ++sl) wait_row(p, slot_entry(st, p.idx, sl, i), st);
    if (st.var_off >= 0)
      for (int w = __ldg(p.idx + st.var_off + i); w < __ldg(p.idx + st.var_off + i + 1); ++w) wait_row(p, __ldg(p.idx + w), st);
    const bool act = j < h;
    const int jj = act ? j : 0;
    float z[5];
#pragma unroll
    for (int g = 0; g < 5; ++g) z[g] = (g < G) ? bias[g * h + jj] : 0.f;
    for (int s = 0; s < NS; ++s) {
      const T *a = segment_row<T>(p, st, s, i);
      const T *wk = Wt + static_cast<size_t>(s) * h * ldw + jj;
      for (int k = 0; k < h; ++k) {
        const float av = to_f<T>(__ldcg(a + k));
#pragma unroll
        for (int g = 0; g < 5; ++g)
          if (g < G) z[g] = fmaf(av, to_f<T>(wk[static_cast<size_t>(k) * ldw + g * h]), z[g]);
      }
    }
    if (act) cell_epilogue<T>(p, st, i, j, z);
    __syncwarp();
    if (lane == 0) publish_row(p, st.out_row0 + i, min(32, h - (j - lane)));
  }
}

// Output linear O (y = W h + b, fp32 logits), fp32 path: warp per row, W fp32 [C x h].
template <typename T>
__device__ void simt_linear_out(const KParams &p, const DevStep &st) {
  const int h = p.hidden;
  const DevWeightSet &w = p.w[st.wset];
  const float *W = static_cast<const float *>(step_W(p, st));
  const float *bias = step_b(p, st);
  const int C = st.gates;  // logits of this step (out_dim of its op type)
  const int lane = threadIdx.x & 31;
  const long gw = (static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const long nw = (static_cast<long>(gridDim.x) * blockDim.x) >> 5;
  float bv[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) bv[c] = c < C ? __ldg(bias + c) : 0.f;
  for (long i = gw; i < st.m; i += nw) {
    const int e = slot_entry(st, p.idx, 0, static_cast<int>(i));
    wait_row(p, e, st);
    const T *a = entry_row<T>(p, w, e, false);
    float acc[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) acc[c] = 0.f;
    for (int k = lane; k < h; k += 32) {
      const float av = to_f<T>(__ldcg(a + k));
#pragma unroll
      for (int c = 0; c < 16; ++c)
        if (c < C) acc[c] = fmaf(av, __ldg(W + c * h + k), acc[c]);
    }
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      float v = acc[c];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      acc[c] = v;
    }
    if (lane == 0) {
      float *y = p.Y + static_cast<size_t>(st.out_row0 + i) * p.ycols;
#pragma unroll
      for (int c = 0; c < 16; ++c)
        if (c < C) y[c] = acc[c] + bv[c];  // sink: no readiness to publish (bias loaded up front)
    }
  }
}

// bf16 path output linear (HBM-bound): one warp, rows i0 and i0+1, W staged in shared memory as
// [c][k] fp32 (or read from global when it does not fit); 16 B row loads (lane owns chunks lane,
// lane+32, ...), h % 64 == 0.
__device__ void linear_out_rows_bf16(const KParams &p, const DevStep &st, long i0, const float *Ws) {
  const int h = p.hidden, C = st.gates;
  const DevWeightSet &w = p.w[st.wset];
  const float *bias = step_b(p, st);
  const int lane = threadIdx.x & 31;
  const int nch = h / 8;                 // 16 B chunks per row
  const int cpl = (nch + 31) / 32;       // chunks per lane (<= 4 for h <= 1024)
  // bias first, all classes at once: loaded inside the store loop below, each class's load waited
  // for the previous class's store (one L2 round trip per class, ~6 us per 24-row item; staging
  // the bias in shared memory does not help: the loads still order behind the stores)
  float bv[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) bv[c] = c < C ? __ldg(bias + c) : 0.f;
  uint4 v[2][4];
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const long i = i0 + r;
    const __nv_bfloat16 *a = nullptr;
    if (i < st.m) {
      const int e = slot_entry(st, p.idx, 0, static_cast<int>(i));
      wait_row(p, e, st);
      a = entry_row<__nv_bfloat16>(p, w, e, false);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int ch = lane + 32 * q;
      v[r][q] = (a != nullptr && q < cpl && ch < nch) ? __ldcg(reinterpret_cast<const uint4 *>(a) + ch)
                                                       : make_uint4(0, 0, 0, 0);
    }
  }
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    float acc[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) acc[c] = 0.f;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int ch = lane + 32 * q;
      if (q >= cpl || ch >= nch) continue;
      const __nv_bfloat16 *e = reinterpret_cast<const __nv_bfloat16 *>(&v[r][q]);
      float av[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) av[u] = __bfloat162float(e[u]);
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        if (c >= C) break;
        const float4 w0 = *reinterpret_cast<const float4 *>(Ws + c * h + ch * 8);
        const float4 w1 = *reinterpret_cast<const float4 *>(Ws + c * h + ch * 8 + 4);
        acc[c] = fmaf(av[0], w0.x, fmaf(av[1], w0.y, fmaf(av[2], w0.z, fmaf(av[3], w0.w, acc[c]))));
        acc[c] = fmaf(av[4], w1.x, fmaf(av[5], w1.y, fmaf(av[6], w1.z, fmaf(av[7], w1.w, acc[c]))));
      }
    }
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      if (c >= C) break;  // warp-uniform
      float x = acc[c];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      acc[c] = x;
    }
    const long i = i0 + r;
    if (lane == 0 && i < st.m) {
      float *y = p.Y + static_cast<size_t>(st.out_row0 + i) * p.ycols;
#pragma unroll
      for (int c = 0; c < 16; ++c)
        if (c < C) y[c] = acc[c] + bv[c];  // sink: no readiness to publish (bias loaded up front)
    }
  }
}

// ------------------------------------------------------------------------------------------------
// MV-RNN (Socher et al. 2012; Table 4).  Node matrices are stored transposed: the Mx
// block of a node (and every word matrix of the packed table) holds M^T, row-major h x h.
// ------------------------------------------------------------------------------------------------
// Matrix of operand entry e: a node record (Mx) or a word matrix of the packed table.
template <typename T>
__device__ __forceinline__ const T *mv_matrix(const KParams &p, const DevStep &st, int e) {
  const size_t hh = static_cast<size_t>(p.hidden) * p.hidden;
  return e >= 0 ? static_cast<const T *>(p.Mx) + static_cast<size_t>(e) * hh
                : static_cast<const T *>(p.w[st.wset].mat) + static_cast<size_t>(-1 - e) * hh;
}

// Matvec step u = [B a; A b] -> U (HBM-bound: every item streams one h x h matrix once).
// Item t (one CTA): member i = t / 2, half q = t % 2; q = 0: B a (matrix of slot 1, vector of slot
// 0) -> U[:, 0:h]; q = 1: A b -> U[:, h:2h].  (M x)[c] = sum_k M^T[k][c] x[k]: thread (rg, cg) owns
// VEC columns and a strided set of rows k; partial sums are reduced through shared memory.
// svec: h floats; sred: blockDim.x * VEC floats.
template <typename T>
__device__ void mv_vec_items(const KParams &p, const DevStep &st, int t_begin, int t_step, float *svec, float *sred) {
  constexpr int VEC = 16 / sizeof(T);
  const int h = p.hidden, nthr = blockDim.x, tid = threadIdx.x;
  const int ncg = h / VEC;
  const int nrg = ncg <= nthr ? nthr / ncg : 1;
  const int T_ = 2 * st.m;
  T *U = static_cast<T *>(p.U);
  for (int t = t_begin; t < T_; t += t_step) {
    const int i = t >> 1, q = t & 1;
    const int ev = slot_entry(st, p.idx, q, i);      // vector: a (q = 0) or b (q = 1)
    const int em = slot_entry(st, p.idx, 1 - q, i);  // matrix: B (q = 0) or A (q = 1)
    wait_row(p, ev, st);
    wait_row(p, em, st);
    const T *vec = entry_row<T>(p, p.w[st.wset], ev, false);
    const T *Mt = mv_matrix<T>(p, st, em);
    for (int k = tid; k < h; k += nthr) svec[k] = to_f<T>(__ldcg(vec + k));
    __syncthreads();
    T *dst = U + (static_cast<size_t>(st.out_row0 + i) * 2 + q) * h;
    for (int cg0 = 0; cg0 < ncg; cg0 += nthr) {  // one pass unless h > nthr * VEC
      const int rg = ncg <= nthr ? tid / ncg : 0;
      const int cg = ncg <= nthr ? tid % ncg : cg0 + tid;
      float acc[VEC];
#pragma unroll
      for (int e = 0; e < VEC; ++e) acc[e] = 0.f;
      if (rg < nrg && cg < ncg) {
        const uint4 *col = reinterpret_cast<const uint4 *>(Mt + static_cast<size_t>(cg) * VEC);
        const size_t ld = static_cast<size_t>(h) / VEC;  // uint4 per matrix row
        int k = rg;
        for (; k + 3 * nrg < h; k += 4 * nrg) {
          uint4 v[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) v[u] = __ldcg(col + static_cast<size_t>(k + u * nrg) * ld);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const T *e = reinterpret_cast<const T *>(&v[u]);
            const float x = svec[k + u * nrg];
#pragma unroll
            for (int c = 0; c < VEC; ++c) acc[c] = fmaf(to_f<T>(e[c]), x, acc[c]);
          }
        }
        for (; k < h; k += nrg) {
          const uint4 v = __ldcg(col + static_cast<size_t>(k) * ld);
          const T *e = reinterpret_cast<const T *>(&v);
          const float x = svec[k];
#pragma unroll
          for (int c = 0; c < VEC; ++c) acc[c] = fmaf(to_f<T>(e[c]), x, acc[c]);
        }
      }
      if (nrg == 1) {
        if (cg < ncg)
#pragma unroll
          for (int c = 0; c < VEC; ++c) dst[cg * VEC + c] = from_f<T>(acc[c]);
      } else {
        if (rg < nrg)
#pragma unroll
          for (int c = 0; c < VEC; ++c) sred[rg * h + cg * VEC + c] = acc[c];
        __syncthreads();
        for (int c = tid; c < h; c += nthr) {
          float sum = 0.f;
          for (int r = 0; r < nrg; ++r) sum += sred[r * h + c];
          dst[c] = from_f<T>(sum);
        }
      }
    }
    asm volatile("fence.proxy.async.global;" ::: "memory");  // U is read by TMA in the p step
    __threadfence();
    __syncthreads();  // svec / sred reused; every store of the item precedes the publication
    if (tid == 0) publish_row(p, st.out_row0 + i, h / 2);
  }
}

// fp32 path of the matrix product: P^T[r][j] = sum_k [A^T | B^T][r][k] W_M[j][k] (Wt = W_M^T
// [2h][h]); warp task = (matrix row R of the batch's m * h rows, 32 columns).
template <typename T>
__device__ void simt_mv_mat(const KParams &p, const DevStep &st) {
  const int h = p.hidden;
  const T *Wt = static_cast<const T *>(step_W(p, st));
  const int lane = threadIdx.x & 31;
  const int nub = (h + 31) / 32;
  const long tasks = static_cast<long>(st.m) * h * nub;
  const long gw = (static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const long nw = (static_cast<long>(gridDim.x) * blockDim.x) >> 5;
  T *Mx = static_cast<T *>(p.Mx);
  for (long task = gw; task < tasks; task += nw) {
    const long R = task / nub;
    const int i = static_cast<int>(R / h), r = static_cast<int>(R % h);
    const int j = static_cast<int>(task % nub) * 32 + lane;
    const int e0 = slot_entry(st, p.idx, 0, i), e1 = slot_entry(st, p.idx, 1, i);
    wait_row(p, e0, st);
    wait_row(p, e1, st);
    const int jj = j < h ? j : 0;
    float z = 0.f;
    for (int sg = 0; sg < 2; ++sg) {
      const T *a = mv_matrix<T>(p, st, sg == 0 ? e0 : e1) + static_cast<size_t>(r) * h;
      const T *wk = Wt + static_cast<size_t>(sg) * h * h + jj;
      for (int k = 0; k < h; ++k) z = fmaf(to_f<T>(__ldcg(a + k)), to_f<T>(wk[static_cast<size_t>(k) * h]), z);
    }
    if (j < h) Mx[(static_cast<size_t>(st.out_row0 + i) * h + r) * h + j] = from_f<T>(z);
    __syncwarp();
    if (lane == 0) publish_row(p, st.out_row0 + i, min(32, h - (j - lane)));
  }
}

// ------------------------------------------------------------------------------------------------
// fp32 persistent kernel: all SIMT
// ------------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads, 1) ed_persistent_f32(const __grid_constant__ KParams p) {
  __shared__ float s_vec[2048];          // MV-RNN matvec operand (h <= 2048)
  __shared__ float s_red[kThreads * 4];  // MV-RNN partial sums
  prologue_checks<float>(p);
  if (blockIdx.x == 0 && threadIdx.x == 0) p.ts[0] = globaltimer();
  for (int s = 0; s < p.num_steps; ++s) {  // dataflow: tasks wait on their input rows, no barrier
    const DevStep st = p.steps[s];
    if (st.cell == ED_CELL_LINEAR_OUT || st.cell == kCellTaggerOut)
      simt_linear_out<float>(p, st);
    else if (st.cell == ED_CELL_MVRNN_INTERNAL)
      mv_vec_items<float>(p, st, blockIdx.x, gridDim.x, s_vec, s_red);
    else if (st.cell == kCellMvMat)
      simt_mv_mat<float>(p, st);
    else
      simt_gemm_step<float>(p, st);
    __syncthreads();
    if (threadIdx.x == 0) stamp_step(p, s);
  }
}

// ------------------------------------------------------------------------------------------------
// bf16 persistent kernel: tcgen05 tensor-core engine
// ------------------------------------------------------------------------------------------------
struct Pipe {
  uint32_t it = 0;  // global K-chunk counter (stage = it % kStages, phase = (it / kStages) & 1)
  uint32_t ti = 0;  // global tile counter (accumulator = ti & 1)
};

__device__ __forceinline__ bool is_umma_cell(int cell) {
  return cell == ED_CELL_LINEAR_OUT || cell == ED_CELL_TREELSTM_LEAF || cell == ED_CELL_TREELSTM_INTERNAL || cell == ED_CELL_TREEGRU_LEAF ||
         cell == ED_CELL_TREEGRU_INTERNAL || cell == ED_CELL_TREEFC_INTERNAL || cell == ED_CELL_LSTM ||
         cell == ED_CELL_LATTICE_CHAR || cell == ED_CELL_LATTICE_WORD || cell == kCellLatticeLink ||
         cell == ED_CELL_LATTICEGRU_CHAR || cell == ED_CELL_LATTICEGRU_WORD ||
         cell == ED_CELL_TAGGER || cell == kCellMvP || cell == kCellMvMat;
}

// Per-cell configuration of the tensor-core epilogue: G gates, U units per column tile (must
// match ed::cell_units; N = G*U <= 256), NAUX fp32 rows of C read per member (children / previous state).
// Per-cell configuration of the tensor-core epilogue: G gates, U units per column tile (must
// match ed::cell_units; N = G*U <= 256), NC fp32 C rows and NH bf16 H rows read per member
// (children / previous state), prefetched one 8-unit step ahead.
template <int CELL> struct CellCfg;
template <> struct CellCfg<ED_CELL_TREELSTM_LEAF> { static constexpr int G = 3, U = 80, NC = 0, NH = 0; };
template <> struct CellCfg<ED_CELL_TREELSTM_INTERNAL> { static constexpr int G = 5, U = 48, NC = 2, NH = 0; };
template <> struct CellCfg<ED_CELL_TREEGRU_LEAF> { static constexpr int G = 2, U = 128, NC = 0, NH = 0; };
template <> struct CellCfg<ED_CELL_TREEGRU_INTERNAL> { static constexpr int G = 5, U = 48, NC = 0, NH = 2; };
template <> struct CellCfg<ED_CELL_TREEFC_INTERNAL> { static constexpr int G = 1, U = 256, NC = 0, NH = 0; };
template <> struct CellCfg<ED_CELL_LSTM> { static constexpr int G = 4, U = 64, NC = 1, NH = 0; };
template <> struct CellCfg<ED_CELL_LATTICE_CHAR> { static constexpr int G = 4, U = 64, NC = 1, NH = 0; };
template <> struct CellCfg<ED_CELL_LATTICE_WORD> { static constexpr int G = 3, U = 80, NC = 1, NH = 0; };
template <> struct CellCfg<ED_CELL_LATTICEGRU_CHAR> { static constexpr int G = 4, U = 64, NC = 0, NH = 1; };
template <> struct CellCfg<ED_CELL_LATTICEGRU_WORD> { static constexpr int G = 4, U = 64, NC = 0, NH = 1; };
template <> struct CellCfg<kCellLatticeLink> { static constexpr int G = 1, U = 256, NC = 0, NH = 0; };
template <> struct CellCfg<ED_CELL_TAGGER> { static constexpr int G = 1, U = 256, NC = 0, NH = 0; };
template <> struct CellCfg<kCellMvP> { static constexpr int G = 1, U = 256, NC = 0, NH = 0; };

// Hidden units of column tile ct (the last tile of a row may be narrower: h need not divide by U).
__device__ __forceinline__ int tile_units(const DevStep &st, int h, int ct) { return min(st.units, h - ct * st.units); }
// MMA N of a column tile: G * units, or 16 for the output linear (C <= 16 classes, zero-padded W_O)
__device__ __forceinline__ int tile_cols(const DevStep &st, int h, int ct) {
  return st.cell == ED_CELL_LINEAR_OUT ? 16 : st.gates * tile_units(st, h, ct);
}

__device__ __forceinline__ float f4get(const float4 &v, int k) {
  return k == 0 ? v.x : (k == 1 ? v.y : (k == 2 ? v.z : v.w));
}
__device__ __forceinline__ void unpack_bf16x8(const uint4 &v, float *out) {
  const __nv_bfloat162 *p = reinterpret_cast<const __nv_bfloat162 *>(&v);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float2 f = __bfloat1622float2(p[q]);
    out[2 * q] = f.x;
    out[2 * q + 1] = f.y;
  }
}

// Epilogue of one 128 x (G*units) tile for thread r (= TMEM lane = tile row): wait for the
// accumulator, then per 8 units: tcgen05.ld -> gates (fp32, MUFU tanh.approx) -> vector stores.
// Child / previous-state rows of the next 8-unit step are prefetched while the current one is
// processed; bias comes from shared memory.
// Split-K pair exchange of one tile (rank < 0: the step is not split).  Rank r of the CTA pair
// holds the partial sums of K half r for all 16 units of the tile and finalises the 8-unit half r:
// it sends the other half's partials (G x 8 fp32 per row) into the partner's receive buffer with
// st.async (complete_tx on the partner's xfull) once the partner has signalled xfree.
struct XCtx {
  int rank;             // cluster rank (0 / 1), or -1
  uint32_t par;         // phase parity of xfull / xfree for this tile
  uint64_t *xfree;      // local: the partner may write its buffer (partner arrives remotely)
  uint64_t *xfull;      // local: the partner's partials have landed in recv
  uint32_t rrecv;       // cluster address of the partner's receive buffer
  uint32_t rxfull;      // cluster address of the partner's xfull
  const float *recv;    // local receive buffer: float4 (q, row) at (q * 128 + row) * 4
};

template <int CELL, bool SPLIT = false>
__device__ __forceinline__ void umma_epilogue(const KParams &p, const DevStep &st, uint32_t tacc, uint64_t *tfull_bar,
                                              uint32_t parity, int row_tile, int col_tile, int r,
                                              const float *sbias, bool bias_smem, const XCtx &x,
                                              unsigned long long *tr = nullptr) {
  using CC = CellCfg<CELL>;
  constexpr int G = CC::G, NC = CC::NC, NH = CC::NH;
  const int h = p.hidden;
  const int i = row_tile * kTileM + r;
  const bool valid = i < st.m;
  const int jb = col_tile * st.units;
  const int ngroups = tile_units(st, h, col_tile) / 16;
  int e0 = p.zero_row, e1 = p.zero_row;
  if (valid && st.nslots > 0) e0 = slot_entry(st, p.idx, 0, i);
  if (valid && st.nslots > 1) e1 = slot_entry(st, p.idx, 1, i);
  if (e0 < 0) e0 = p.zero_row;  // external inputs have no c / h record here
  if (e1 < 0) e1 = p.zero_row;
  if (valid && !(row_ready(p, e0, st) && row_ready(p, e1, st))) {  // acquire the rows read below
    wait_row(p, e0, st);
    wait_row(p, e1, st);
  }
  const float4 *cp0 = reinterpret_cast<const float4 *>(p.C + static_cast<size_t>(e0) * h + jb);
  const float4 *cp1 = reinterpret_cast<const float4 *>(p.C + static_cast<size_t>(e1) * h + jb);
  const __nv_bfloat16 *Hb = static_cast<const __nv_bfloat16 *>(p.H);
  int dbeg = 0, dend = 0;  // copies of this result row (staged operand rows, instance output)
  __nv_bfloat16 *cpy0 = nullptr, *cpy1 = nullptr;  // the first two copies' rows, resolved up front
  if (valid && CELL != kCellLatticeLink) {
    dbeg = __ldg(p.dst_off + st.out_row0 + i);
    dend = __ldg(p.dst_off + st.out_row0 + i + 1);
    if (dbeg < dend) cpy0 = copy_row<__nv_bfloat16>(p, __ldg(p.idx + dbeg++));
    if (dbeg < dend) cpy1 = copy_row<__nv_bfloat16>(p, __ldg(p.idx + dbeg++));
  }
  const uint4 *hp0 = reinterpret_cast<const uint4 *>(Hb + static_cast<size_t>(e0) * h + jb);
  const uint4 *hp1 = reinterpret_cast<const uint4 *>(Hb + static_cast<size_t>(e1) * h + jb);
  // lattice char: words ending here (variadic inputs)
  int wbeg = 0, wend = 0;
  if constexpr (CELL == ED_CELL_LATTICE_CHAR || CELL == ED_CELL_LATTICEGRU_CHAR) {
    if (valid) {
      wbeg = __ldg(p.idx + st.var_off + i);
      wend = __ldg(p.idx + st.var_off + i + 1);
      for (int w = wbeg; w < wend; ++w) wait_row(p, __ldg(p.idx + w), st);  // words ending here (c^w, l_w)
    }
  }
  // Child / previous-state rows are prefetched two 8-unit passes ahead (passes are processed in
  // pairs, each with its own register buffer): both passes of a 16-unit tile are loaded before the
  // accumulator wait, so the tail steps' epilogue has no L2 round trip inside the pass loop.
  const int nsteps = ngroups * 2;  // even
  float4 cbuf[2][NC > 0 ? 2 * NC : 1];
  uint4 hbuf[2][NH > 0 ? NH : 1];
#pragma unroll
  for (int b2 = 0; b2 < 2; ++b2) {
#pragma unroll
    for (int q = 0; q < NC; ++q) ldcg_v8((q == 0 ? cp0 : cp1) + b2 * 2, cbuf[b2][2 * q], cbuf[b2][2 * q + 1]);
  }
#pragma unroll
  for (int q = 0; q < NH; ++q) ldcg_v8(q == 0 ? hp0 : hp1, hbuf[0][q], hbuf[1][q]);  // both halves of pair 0
#if ED_EPI_WAIT_SLEEP > 0
  mbar_wait_sleep(tfull_bar, parity, ED_EPI_WAIT_SLEEP);
#else
  mbar_wait_warp(tfull_bar, parity);
#endif
  tc_fence_after();
  if (tr != nullptr && r == 0) *tr = globaltimer();
  __nv_bfloat16 *H = static_cast<__nv_bfloat16 *>(p.H);
  const size_t orow = static_cast<size_t>(st.out_row0 + (valid ? i : 0));
  // A warp whose 32 rows all lie past m skips the pass loop: tcgen05.ld bandwidth (~64 B/clk per
  // SM) is shared by the four epilogue warps, so small-m tail tiles read TMEM for their live rows only.
  const bool warp_live = row_tile * kTileM + (r & ~31) < st.m;
  if (SPLIT && warp_live) {
    // split-K: send the partner's 8-unit half of this row's partial sums, then wait for ours
    float zs[G][8];
#pragma unroll
    for (int g = 0; g < G; ++g) tmem_ld8(tacc + static_cast<uint32_t>(g * 16 + (x.rank ^ 1) * 8), zs[g]);
    tmem_wait_ld();
#ifdef ED_SPLIT_TRACE
    if (tr != nullptr && r == 0) tr[8] = globaltimer();
#endif
    mbar_wait_cluster(x.xfree, x.par);
#ifdef ED_SPLIT_TRACE
    if (tr != nullptr && r == 0) tr[9] = globaltimer();
#endif
#pragma unroll
    for (int g = 0; g < G; ++g)
#pragma unroll
      for (int q = 0; q < 2; ++q)
        st_async_v4(x.rrecv + static_cast<uint32_t>(((2 * g + q) * kTileM + r) * 16), zs[g][4 * q], zs[g][4 * q + 1],
                    zs[g][4 * q + 2], zs[g][4 * q + 3], x.rxfull);
#ifdef ED_SPLIT_TRACE
    if (tr != nullptr && r == 0) tr[10] = globaltimer();
#endif
    mbar_wait_cluster(x.xfull, x.par);
#ifdef ED_SPLIT_TRACE
    if (tr != nullptr && r == 0) tr[11] = globaltimer();
#endif
  }
#pragma unroll 1
  for (int sp0 = 0; sp0 < (warp_live ? nsteps : 0); sp0 += 2) {
  uint4 hlo = make_uint4(0, 0, 0, 0);  // bf16 h of the pair's first half, stored with the second
#pragma unroll
  for (int b2 = 0; b2 < 2; ++b2) {
    if (SPLIT && b2 != x.rank) continue;  // split-K: the partner finalises this half
    const int sp = sp0 + b2;
    const int gq = sp >> 1, half = sp & 1;
    float4 cc[NC > 0 ? 2 * NC : 1];
    uint4 hc[NH > 0 ? NH : 1];
#pragma unroll
    for (int q = 0; q < 2 * NC; ++q) cc[q] = cbuf[b2][q];
#pragma unroll
    for (int q = 0; q < NH; ++q) hc[q] = hbuf[b2][q];
    if (sp + 2 < nsteps) {
#pragma unroll
      for (int q = 0; q < NC; ++q) ldcg_v8((q == 0 ? cp0 : cp1) + (sp + 2) * 2, cbuf[b2][2 * q], cbuf[b2][2 * q + 1]);
      if (b2 == 1) {  // the next pair's h, both halves in one 32 B load
#pragma unroll
        for (int q = 0; q < NH; ++q) ldcg_v8((q == 0 ? hp0 : hp1) + sp0 + 2, hbuf[0][q], hbuf[1][q]);
      }
    }
    float z[G][8];
#pragma unroll
    for (int g = 0; g < G; ++g) tmem_ld8(tacc + static_cast<uint32_t>(gq * G * 16 + g * 16 + half * 8), z[g]);
    tmem_wait_ld();
    if (SPLIT) {  // + the partner's partial sums of K half (rank ^ 1)
#pragma unroll
      for (int g = 0; g < G; ++g)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const float4 v = lds_f4(x.recv + ((2 * g + q) * kTileM + r) * 4);
          z[g][4 * q] += v.x; z[g][4 * q + 1] += v.y; z[g][4 * q + 2] += v.z; z[g][4 * q + 3] += v.w;
        }
    }
    if (tr != nullptr && r == 0 && sp < 2) tr[4 + 2 * sp] = globaltimer();
    if (!valid) continue;
    const int j0 = jb + sp * 8;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      // explicit state spaces: a generic load of the shared bias would be ordered behind this
      // thread's outstanding global stores of the previous pass (an L2 round trip per pass)
      float4 b0, b1;
      if (bias_smem) {
        b0 = lds_f4(sbias + g * h + j0);
        b1 = lds_f4(sbias + g * h + j0 + 4);
      } else {
        b0 = __ldg(reinterpret_cast<const float4 *>(sbias + g * h + j0));
        b1 = __ldg(reinterpret_cast<const float4 *>(sbias + g * h + j0 + 4));
      }
      z[g][0] += b0.x; z[g][1] += b0.y; z[g][2] += b0.z; z[g][3] += b0.w;
      z[g][4] += b1.x; z[g][5] += b1.y; z[g][6] += b1.z; z[g][7] += b1.w;
    }
    constexpr bool HAS_C = !(CELL == ED_CELL_TREEGRU_LEAF || CELL == ED_CELL_TREEGRU_INTERNAL ||
                             CELL == ED_CELL_TREEFC_INTERNAL || CELL == ED_CELL_TAGGER || CELL == kCellMvP ||
                             CELL == ED_CELL_LATTICEGRU_CHAR || CELL == ED_CELL_LATTICEGRU_WORD);
    constexpr bool HAS_H = CELL != kCellLatticeLink;
    float hv[8] = {}, cv[8] = {};
    float hl[8], hr[8];
    if constexpr (NH >= 1) unpack_bf16x8(hc[0], hl);
    if constexpr (NH >= 2) unpack_bf16x8(hc[NH - 1], hr);
    float aux0[8], aux1[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      aux0[k] = NC >= 1 ? f4get(cc[(k >> 2) % (2 * (NC > 0 ? NC : 1))], k & 3) : 0.f;
      aux1[k] = NC >= 2 ? f4get(cc[(2 + (k >> 2)) % (2 * (NC > 0 ? NC : 1))], k & 3) : 0.f;
    }
    if constexpr (CELL == ED_CELL_LATTICE_CHAR) {
      // c = sum_w alpha_w c^w + alpha_e tanh(g), alpha = softmax over {s(i)} U {l_w} (A-23); else LSTM
      float den[8], num[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float si = sigm_fast(z[0][k]);
        const float ei = __expf(si);
        den[k] = ei;
        num[k] = ei * tanh_fast(z[3 % G][k]);
      }
      for (int w = wbeg; w < wend; ++w) {
        const int wr = __ldg(p.idx + w);
        const float4 *xl = reinterpret_cast<const float4 *>(p.X + static_cast<size_t>(wr) * h + j0);
        const float4 *xc = reinterpret_cast<const float4 *>(p.C + static_cast<size_t>(wr) * h + j0);
        const float4 l0 = __ldcg(xl), l1 = __ldcg(xl + 1), c0 = __ldcg(xc), c1 = __ldcg(xc + 1);
        const float lw[8] = {l0.x, l0.y, l0.z, l0.w, l1.x, l1.y, l1.z, l1.w};
        const float cw[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float el = __expf(lw[k]);
          den[k] += el;
          num[k] += el * cw[k];
        }
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        cv[k] = wend > wbeg ? __fdividef(num[k], den[k])
                            : sigm_fast(z[1 % G][k]) * aux0[k] + sigm_fast(z[0][k]) * tanh_fast(z[3 % G][k]);
        hv[k] = sigm_fast(z[2 % G][k]) * tanh_fast(cv[k]);
      }
    } else {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if constexpr (CELL == ED_CELL_TREELSTM_LEAF) {  // [i;o;u]
          cv[k] = sigm_fast(z[0][k]) * tanh_fast(z[2 % G][k]);
          hv[k] = sigm_fast(z[1 % G][k]) * tanh_fast(cv[k]);
        } else if constexpr (CELL == ED_CELL_TREELSTM_INTERNAL) {  // [i;f_l;f_r;o;u]
          cv[k] = sigm_fast(z[0][k]) * tanh_fast(z[4 % G][k]) + sigm_fast(z[1 % G][k]) * aux0[k] +
                  sigm_fast(z[2 % G][k]) * aux1[k];
          hv[k] = sigm_fast(z[3 % G][k]) * tanh_fast(cv[k]);
        } else if constexpr (CELL == ED_CELL_LSTM) {  // [i;f;g;o]
          cv[k] = sigm_fast(z[1 % G][k]) * aux0[k] + sigm_fast(z[0][k]) * tanh_fast(z[2 % G][k]);
          hv[k] = sigm_fast(z[3 % G][k]) * tanh_fast(cv[k]);
        } else if constexpr (CELL == ED_CELL_TREEGRU_LEAF) {  // [z;n]
          hv[k] = (1.f - sigm_fast(z[0][k])) * tanh_fast(z[1 % G][k]);
        } else if constexpr (CELL == ED_CELL_TREEGRU_INTERNAL) {  // [z;r_l;r_r;a_l;a_r]
          const float n = tanh_fast(sigm_fast(z[1 % G][k]) * z[3 % G][k] + sigm_fast(z[2 % G][k]) * z[4 % G][k]);
          const float zz = sigm_fast(z[0][k]);
          hv[k] = (1.f - zz) * n + zz * (hl[k] + hr[k]);
        } else if constexpr (CELL == ED_CELL_TREEFC_INTERNAL) {
          hv[k] = tanh_fast(z[0][k]);
        } else if constexpr (CELL == ED_CELL_LATTICE_WORD) {  // [i;f;g] -> c^w (fp32 C) and bf16 copy in H
          cv[k] = sigm_fast(z[1 % G][k]) * aux0[k] + sigm_fast(z[0][k]) * tanh_fast(z[2 % G][k]);
          hv[k] = cv[k];
        } else if constexpr (CELL == kCellLatticeLink) {  // l = s(.) -> X
          cv[k] = sigm_fast(z[0][k]);
        } else if constexpr (CELL == ED_CELL_LATTICEGRU_CHAR || CELL == ED_CELL_LATTICEGRU_WORD) {
          // GRU (A-27): [r; z; n_x; n_h]; n = tanh(n_x + r * n_h); h = (1 - z) n + z h_prev
          const float rr = sigm_fast(z[0][k]), zz = sigm_fast(z[1 % G][k]);
          const float n = tanh_fast(z[2 % G][k] + rr * z[3 % G][k]);
          hv[k] = (1.f - zz) * n + zz * hl[k];
        } else {  // tagger hidden t = tanh(.), MV-RNN p = tanh(.) -> H
          hv[k] = tanh_fast(z[0][k]);
        }
      }
    }
    if constexpr (CELL == ED_CELL_LATTICEGRU_CHAR) {  // max-pool with the states of words ending here
      for (int w = wbeg; w < wend; ++w) {
        const int wr = __ldg(p.idx + w);
        float hw[8];
        unpack_bf16x8(__ldcg(reinterpret_cast<const uint4 *>(Hb + static_cast<size_t>(wr) * h + j0)), hw);
#pragma unroll
        for (int k = 0; k < 8; ++k) hv[k] = fmaxf(hv[k], hw[k]);
      }
    }
    if constexpr (HAS_H) {
      uint32_t packed[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        __nv_bfloat162 t = __floats2bfloat162_rn(hv[2 * k], hv[2 * k + 1]);
        packed[k] = *reinterpret_cast<uint32_t *>(&t);
      }
      const uint4 hv4 = make_uint4(packed[0], packed[1], packed[2], packed[3]);
      // the pair's two 8-unit halves are one 32 B run of the row: one 256-bit store per row and copy
      // (full L2 sectors instead of two half-sector writes)
      if (SPLIT) {  // split-K: one 8-unit half per CTA, 16 B per row and copy
        st_v4_b32(H + orow * h + j0, hv4);
        if (cpy0 != nullptr) st_v4_b32(cpy0 + j0, hv4);
        if (cpy1 != nullptr) st_v4_b32(cpy1 + j0, hv4);
        for (int d = dbeg; d < dend; ++d) {
          __nv_bfloat16 *dst = copy_row<__nv_bfloat16>(p, __ldg(p.idx + d));
          if (dst != nullptr) st_v4_b32(dst + j0, hv4);
        }
      } else if (b2 == 0) {
        hlo = hv4;
      } else {
        const int jp = j0 - 8;
        st_v8_b32(H + orow * h + jp, hlo, hv4);
        if (cpy0 != nullptr) st_v8_b32(cpy0 + jp, hlo, hv4);
        if (cpy1 != nullptr) st_v8_b32(cpy1 + jp, hlo, hv4);
        for (int d = dbeg; d < dend; ++d) {
          __nv_bfloat16 *dst = copy_row<__nv_bfloat16>(p, __ldg(p.idx + d));
          if (dst != nullptr) st_v8_b32(dst + jp, hlo, hv4);
        }
      }
    }
    if constexpr (HAS_C) {
      float *dst = (CELL == kCellLatticeLink) ? p.X : p.C;
      st_v8_f32(dst + orow * h + j0, cv);  // 8 fp32 = one 32 B sector
    }
    if (tr != nullptr && r == 0 && sp < 2) tr[5 + 2 * sp] = globaltimer();
  }
  }
  if (tr != nullptr && r == 0) tr[1] = globaltimer();
  if (valid) {
    asm volatile("fence.proxy.async.global;" ::: "memory");  // rows may be read by TMA (async proxy)
    if (tr != nullptr && r == 0) tr[2] = globaltimer();
    publish_row(p, static_cast<int>(orow), SPLIT ? 8 : ngroups * 16);
    if (tr != nullptr && r == 0) tr[3] = globaltimer();
  }
}

// Epilogue of one 128-row tile of the output linear y = W_O h + b (fp32 logits, a sink: nothing
// reads Y, so nothing is published): tcgen05.ld of the 16 accumulator columns, bias, C stores.
__device__ __forceinline__ void linear_out_epilogue(const KParams &p, const DevStep &st, uint32_t tacc, uint64_t *tfull_bar,
                                                    uint32_t parity, int row_tile, int r) {
  const int i = row_tile * kTileM + r;
  const int C = st.units;
  const float *bias = step_b(p, st);
  float bv[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) bv[c] = c < C ? __ldg(bias + c) : 0.f;
  mbar_wait(tfull_bar, parity);
  tc_fence_after();
  float v[16];
  tmem_ld16(tacc, v);
  tmem_wait_ld();
  if (i >= st.m) return;
  float *y = p.Y + static_cast<size_t>(st.out_row0 + i) * p.ycols;
#pragma unroll
  for (int c = 0; c < 16; ++c)
    if (c < C) y[c] = v[c] + bv[c];
}

// Epilogue of one 128 x units tile of the MV-RNN matrix product: rows R = row_tile * 128 + r of the
// batch's m * h rows of P^T (node i = R / h, matrix row R % h), stored bf16 into the node's Mx block.
// A warp's 32 rows belong to one node (h % 64 == 0): lane 0 publishes 32 x units elements.
__device__ __forceinline__ void mv_mat_epilogue(const KParams &p, const DevStep &st, uint32_t tacc, uint64_t *tfull_bar,
                                                uint32_t parity, int row_tile, int col_tile, int r) {
  const int h = p.hidden;
  const long R = static_cast<long>(row_tile) * kTileM + r;
  const bool valid = R < static_cast<long>(st.m) * h;
  const int i = valid ? static_cast<int>(R / h) : 0, rr = static_cast<int>(R % h);
  const int jb = col_tile * st.units, cols = tile_units(st, h, col_tile);
  __nv_bfloat16 *dst = static_cast<__nv_bfloat16 *>(p.Mx) + (static_cast<size_t>(st.out_row0 + i) * h + rr) * h + jb;
  mbar_wait(tfull_bar, parity);
  tc_fence_after();
#pragma unroll 1
  for (int c0 = 0; c0 < cols; c0 += 32) {
    float v[32];
    tmem_ld16(tacc + static_cast<uint32_t>(c0), v);
    if (c0 + 16 < cols) tmem_ld16(tacc + static_cast<uint32_t>(c0 + 16), v + 16);
    tmem_wait_ld();
    if (!valid) continue;
    const int nc = min(32, cols - c0);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (q * 8 >= nc) break;
      uint32_t pk[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        __nv_bfloat162 t = __floats2bfloat162_rn(v[q * 8 + 2 * k], v[q * 8 + 2 * k + 1]);
        pk[k] = *reinterpret_cast<uint32_t *>(&t);
      }
      *reinterpret_cast<uint4 *>(dst + c0 + q * 8) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
    }
  }
  asm volatile("fence.proxy.async.global;" ::: "memory");  // Mx blocks are read by TMA later
  __threadfence();
  __syncwarp();
  if (valid && (threadIdx.x & 31) == 0) publish_row(p, st.out_row0 + i, 32 * cols);
}

// Work items of a step: tensor-core tiles (row tile x column tile), or SIMT groups of kSimtRows
// rows.  Item t of step s runs on CTA (t + off_s) mod G, off_s = running item count mod G, so
// consecutive (often independent) steps land on different SMs.
constexpr int kSimtRows = 2 * (kThreadsTC / 32);  // every warp of the CTA, 2 rows each
__device__ __forceinline__ int step_items(const DevStep &st, int h) {
  if (st.cell == kCellMvMat) return static_cast<int>((static_cast<long>(st.m) * h + kTileM - 1) / kTileM) * st.n_col_tiles;
  if (st.cell == ED_CELL_MVRNN_INTERNAL) return 2 * st.m;  // matvec: one CTA per (member, half)
  if (is_umma_cell(st.cell)) return ((st.m + kTileM - 1) / kTileM) * st.n_col_tiles * (step_split(st) ? 2 : 1);
  return (st.m + kSimtRows - 1) / kSimtRows;
}
// K chunks per pipeline stage.  One full/empty mbarrier round costs ~0.3 us whatever its payload
// (scripts/loop_probe.cu), so a small tile (m <= 120 rows: A chunk = round8(m) x 128 B) packs
// several K chunks into one 48 KB stage: chunk q's A at q * abytes, its B at kps * abytes + q * N * 128 B.
// M = 128 MMAs read 128 A rows from q * abytes; rows past the tile's m are never stored.
#ifndef ED_KPS_MAX
#define ED_KPS_MAX 4  // measured: 4 beats 1, 2, 3 and 16 on cfg2 / cfg3 / cfg5 (r01t A/B)
#endif
__device__ __forceinline__ int step_kps(const DevStep &st, int kc_total, uint32_t *abytes) {
  if (st.cell == kCellMvMat) { *abytes = kAStage; return 1; }
  const int rows = min(kTileM, (st.m + 7) & ~7);
  *abytes = static_cast<uint32_t>(rows) * 128u;
  const int bb = (st.cell == ED_CELL_LINEAR_OUT ? 16 : st.gates * st.units) * 128;
  // small tiles: the 48 KB stage is cut as [A_0 .. A_{k-1} | B_0 .. B_{k-1}], k = 48 KB / (A + B chunk)
  const int k = *abytes < static_cast<uint32_t>(kAStage) ? kStageBytes / (static_cast<int>(*abytes) + bb) : 1;
  return max(1, min(min(k, kc_total), ED_KPS_MAX));
}
__device__ __forceinline__ int first_item(uint32_t off) {
  return static_cast<int>((blockIdx.x + gridDim.x - off % gridDim.x) % gridDim.x);
}

__global__ void __launch_bounds__(kThreadsTC, 1) ed_persistent_bf16(const __grid_constant__ KParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
#if ED_SMEM_SLACK == 0
  if (smem != smem_raw) __trap();  // built without alignment slack: the base must be 1024-aligned
#endif
  uint8_t *stages = smem;
  const void **rowtab = reinterpret_cast<const void **>(smem + kStages * kStageBytes);  // [2][128][2] row ptrs
  float *sbias = reinterpret_cast<float *>(smem + kStages * kStageBytes + 2 * kRowTab);
  float *swout = reinterpret_cast<float *>(smem + kStages * kStageBytes + 2 * kRowTab + kBiasBytes);
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + kStages * kStageBytes + 2 * kRowTab + kBiasBytes +
                                                kWoutBytes);
  uint64_t *full = bars, *empty = bars + kStages, *tfull = bars + 2 * kStages, *tempty = bars + 2 * kStages + 2;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 2 * kStages + 4);
  uint64_t *xfree = bars + 2 * kStages + 5, *xfull = bars + 2 * kStages + 6;  // split-K pair exchange
  // split-K receive buffer (<= 128 rows x 5 gates x 8 units fp32 = 20 KB): aliases the bias and
  // output-weight buffers, which split steps do not use (their bias is read from L2)
  const float *xrecv = sbias;
  static_assert(kBiasBytes + kWoutBytes >= kTileM * 5 * 8 * 4, "split-K receive buffer");

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(full + s, 2 + kLoaderThreads);  // A TMA-or-nothing + every loader thread's cp.async + B
      mbar_init(empty + s, 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull + a, 1);
      mbar_init(tempty + a, kEpiThreads);
    }
    mbar_init(xfree, 1);
    mbar_init(xfull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 4) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  if (p.has_split) cluster_sync_all();  // the partner's barriers are initialised before any remote arrive
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  prologue_checks<__nv_bfloat16>(p);
#if ED_PREFETCH_TMAP
  if (tid == 192) {  // the operand loaders' descriptors into the TMA descriptor cache
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&p.tm_h128)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&p.tm_u)) : "memory");
  }
#endif
  if (blockIdx.x == 0 && tid == 0) p.ts[0] = globaltimer();

  const int h = p.hidden;
  const int G = static_cast<int>(gridDim.x);
  Pipe pipe;
  uint32_t tab_tile = 0;    // loader threads: row-table buffer toggle
  uint32_t off = 0;         // running item offset (work rotation)

  // Register split per warpgroup (setmaxnreg): the epilogue warpgroup (warps 0-3) keeps the gate
  // math, its prefetched child rows and copy pointers in registers; the MMA issuer, the weight
  // loader and the operand loaders (warps 4-11) need few.  Every role walks the steps in order;
  // there is no grid barrier between steps (dataflow).
  if (warp < 4) {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kEpiRegs));
    uint32_t xcnt = 0;  // split tiles exchanged (xfull / xfree phase)
  for (int s = 0; s < p.num_steps; ++s) {
    const DevStep st = p.steps[s];
    const bool split = step_split(st);
    if (split) {  // pair items (2j, 2j + 1) on the two CTAs of a cluster: even rotation offset
      off = (off + 1u) & ~1u;
      if (off >= static_cast<uint32_t>(G)) off -= static_cast<uint32_t>(G);
    }
    const int T = step_items(st, h);
    const int t0 = first_item(off);
    off = (off + static_cast<uint32_t>(T)) % static_cast<uint32_t>(G);
    if (t0 >= T) continue;  // no work for this CTA in this step
    ED_TRACE(p, s, 0, tid == 0 && t0 == 0);
    if (!is_umma_cell(st.cell)) {
      if (st.cell == ED_CELL_MVRNN_INTERNAL) {  // ---- MV-RNN matvecs: one CTA per item ----
        __syncthreads();  // sbias / swout are free (previous step's epilogue done)
        mv_vec_items<__nv_bfloat16>(p, st, t0, G, sbias, swout);
        if (tid == 0) stamp_step(p, s);
        continue;
      }
      // ---------------- SIMT step (output linear / tagger output): every warp, 2 rows each ----------
      const int C = st.gates;
      const bool in_smem = C * h * 4 <= kWoutBytes;
      if (p.has_split) __syncthreads();  // swout may still hold a split-K exchange of the epilogue
      if (in_smem) {  // 16 B cp.async per piece (no register staging)
        const float *W = static_cast<const float *>(step_W(p, st));
        const uint32_t sw = smem_u32(swout);
        for (int q = tid; q < C * h / 4; q += kThreadsTC) cp_async16(sw + 16u * q, W + 4 * q);
        cp_async_commit();
        cp_async_wait<0>();
      }
      __syncthreads();
      if (p.trace && tid == 0) p.trace[p.num_steps * 64 + blockIdx.x * 4 + 1] = globaltimer();
      const float *Ws = in_smem ? swout : static_cast<const float *>(step_W(p, st));
      for (int t = t0; t < T; t += G) linear_out_rows_bf16(p, st, static_cast<long>(t) * kSimtRows + 2 * warp, Ws);
      if (p.trace && lane == 0) atomicMax(p.trace + p.num_steps * 64 + blockIdx.x * 4 + 2, globaltimer());
      __syncthreads();  // swout is reused by the next SIMT step
      if (tid == 0) stamp_step(p, s);
      continue;
    }
    const int ncols = st.cell == ED_CELL_LINEAR_OUT ? 16 : st.gates * st.units;
    const int kc_total = (cell_segments_dev(st.cell) * h) / kChunkK;
    uint32_t abytes = kAStage;
    const int kc_part = split ? kc_total / 2 : kc_total;  // K chunks per CTA
    const int kps = step_kps(st, kc_part, &abytes);
      // ---------------- epilogue warps ----------------
      const float *bsrc = step_b(p, st);
      const bool bias_smem = !split && bsrc != nullptr && st.cell != ED_CELL_LINEAR_OUT && st.gates * h * 4 <= kBiasBytes;
      if (bias_smem) {  // 16 B cp.async per piece: no register staging, all pieces in flight at once
        const uint32_t sb = smem_u32(sbias);
        for (int q = tid; q < st.gates * h / 4; q += kEpiThreads) cp_async16(sb + 16u * q, bsrc + 4 * q);
        cp_async_commit();
        cp_async_wait<0>();
      }
      asm volatile("bar.sync 2, %0;" ::"n"(kEpiThreads) : "memory");
      const float *bias = bias_smem ? sbias : bsrc;
      for (int t = t0; t < T; t += G) {
        const uint32_t acc = pipe.ti & 1u;
        const uint32_t tacc = tmem_base + (static_cast<uint32_t>(warp * 32) << 16) + acc * 256u;
        const int tile = split ? (t >> 1) : t;
        const int row_tile = tile / st.n_col_tiles, col_tile = tile % st.n_col_tiles;
        const uint32_t par = (pipe.ti >> 1) & 1u;
        XCtx x;
        x.rank = -1;
#ifndef ED_NO_SPLIT
        if (split) {
          // the receive buffer is free once every epilogue thread is past the previous exchange
          asm volatile("bar.sync 2, %0;" ::"n"(kEpiThreads) : "memory");
          const uint32_t crank = static_cast<uint32_t>(t & 1);  // = %cluster_ctarank (even rotation offset)
          x.rank = static_cast<int>(crank);
          x.par = xcnt & 1u;
          ++xcnt;
          x.xfree = xfree;
          x.xfull = xfull;
          x.rrecv = mapa_u32(smem_u32(xrecv), crank ^ 1u);
          x.rxfull = mapa_u32(smem_u32(xfull), crank ^ 1u);
          x.recv = xrecv;
          if (tid == 0) {
            const int live = min(4, (st.m - row_tile * kTileM + 31) / 32);  // warps with rows
            mbar_arrive_tx(xfull, static_cast<uint32_t>(live * 32 * st.gates * 8 * 4));
            mbar_arrive_remote(mapa_u32(smem_u32(xfree), crank ^ 1u));  // the partner may now write our buffer
          }
        }
#endif
#ifndef ED_NO_SPLIT
        if (split) {  // split-K steps (cells of ed::cell_splittable)
          unsigned long long *trp = (p.trace && t == 0) ? p.trace + s * 64 + 6 : nullptr;
          switch (st.cell) {
            case ED_CELL_TREELSTM_INTERNAL:
              umma_epilogue<ED_CELL_TREELSTM_INTERNAL, true>(p, st, tacc, tfull + acc, par, row_tile, col_tile, tid, bias, false, x, trp); break;
            default:
              umma_epilogue<ED_CELL_TREEGRU_INTERNAL, true>(p, st, tacc, tfull + acc, par, row_tile, col_tile, tid, bias, false, x, trp); break;
          }
        } else
#endif
        switch (st.cell) {
          case ED_CELL_TREELSTM_LEAF:
            umma_epilogue<ED_CELL_TREELSTM_LEAF>(p, st, tacc, tfull + acc, par, row_tile, col_tile, tid, bias, bias_smem, x, (p.trace && t == 0) ? p.trace + s * 64 + 6 : nullptr); break;
          case ED_CELL_TREELSTM_INTERNAL:
            umma_epilogue<ED_CELL_TREELSTM_INTERNAL>(p, st, tacc, tfull + acc, par, row_tile, col_tile, tid, bias, bias_smem, x, (p.trace && t == 0) ? p.trace + s * 64 + 6 : nullptr); break;
          case ED_CELL_TREEGRU_LEAF:
            umma_epilogue<ED_CELL_TREEGRU_LEAF>(p, st, tacc, tfull + acc, par, row_tile, col_tile, tid, bias, bias_smem, x, (p.trace && t == 0) ? p.trace + s * 64 + 6 : nullptr); break;
          case ED_CELL_TREEGRU_INTERNAL:
            umma_epilogue<ED_CELL_TREEGRU_INTERNAL>(p, st, tacc, tfull + acc, par, row_tile, col_tile, tid, bias, bias_smem, x, (p.trace && t == 0) ? p.trace + s * 64 + 6 : nullptr); break;
          case ED_CELL_TREEFC_INTERNAL:
            umma_epilogue<ED_CELL_TREEFC_INTERNAL>(p, st, tacc, tfull + acc, par, row_tile, col_tile, tid, bias, bias_smem, x, (p.trace && t == 0) ? p.trace + s * 64 + 6 : nullptr); break;
          case ED_CELL_LSTM:
            umma_epilogue<ED_CELL_LSTM>(p, st, tacc, tfull + acc, par, row_tile, col_tile, tid, bias, bias_smem, x, (p.trace && t == 0) ? p.trace + s * 64 + 6 : nullptr); break;
          case ED_CELL_LATTICE_CHAR:
            umma_epilogue<ED_CELL_LATTICE_CHAR>(p, st, tacc, tfull + acc, par, row_tile, col_tile, tid, bias, bias_smem, x, (p.trace && t == 0) ? p.trace + s * 64 + 6 : nullptr); break;
          case ED_CELL_LATTICEGRU_CHAR:
            umma_epilogue<ED_CELL_LATTICEGRU_CHAR>(p, st, tacc, tfull + acc, par, row_tile, col_tile, tid, bias, bias_smem, x, (p.trace && t == 0) ? p.trace + s * 64 + 6 : nullptr); break;
          case ED_CELL_LATTICEGRU_WORD:
            umma_epilogue<ED_CELL_LATTICEGRU_WORD>(p, st, tacc, tfull + acc, par, row_tile, col_tile, tid, bias, bias_smem, x, (p.trace && t == 0) ? p.trace + s * 64 + 6 : nullptr); break;
          case ED_CELL_LATTICE_WORD:
            umma_epilogue<ED_CELL_LATTICE_WORD>(p, st, tacc, tfull + acc, par, row_tile, col_tile, tid, bias, bias_smem, x, (p.trace && t == 0) ? p.trace + s * 64 + 6 : nullptr); break;
          case kCellLatticeLink:
            umma_epilogue<kCellLatticeLink>(p, st, tacc, tfull + acc, par, row_tile, col_tile, tid, bias, bias_smem, x, (p.trace && t == 0) ? p.trace + s * 64 + 6 : nullptr); break;
          case kCellMvP:
            umma_epilogue<kCellMvP>(p, st, tacc, tfull + acc, par, row_tile, col_tile, tid, bias, bias_smem, x, (p.trace && t == 0) ? p.trace + s * 64 + 6 : nullptr); break;
          case kCellMvMat:
            mv_mat_epilogue(p, st, tacc, tfull + acc, par, row_tile, col_tile, tid); break;
          case ED_CELL_LINEAR_OUT:
            linear_out_epilogue(p, st, tacc, tfull + acc, par, row_tile, tid); break;
          default:
            umma_epilogue<ED_CELL_TAGGER>(p, st, tacc, tfull + acc, par, row_tile, col_tile, tid, bias, bias_smem, x, (p.trace && t == 0) ? p.trace + s * 64 + 6 : nullptr); break;
        }
        ED_TRACE(p, s, 5, tid == 0 && t == 0);
#ifdef ED_LEAF_TRACE  // development: per-CTA end of each of the first step's tiles
        if (p.trace && s == 0 && tid == 0) {
          const int k = (t - t0) / G;
          if (k < 4) p.trace[p.num_steps * 64 + blockIdx.x * 4 + k] = globaltimer();
        }
#endif
        tc_fence_before();
        mbar_arrive(tempty + acc);
        ++pipe.ti;
      }
      asm volatile("bar.sync 2, %0;" ::"n"(kEpiThreads) : "memory");  // sbias reused by the next step
      if (tid == 0) stamp_step(p, s);
  }
  } else {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kProdRegs));
  for (int s = 0; s < p.num_steps; ++s) {
    const DevStep st = p.steps[s];
    const bool split = step_split(st);
    if (split) {  // pair items (2j, 2j + 1) on the two CTAs of a cluster: even rotation offset
      off = (off + 1u) & ~1u;
      if (off >= static_cast<uint32_t>(G)) off -= static_cast<uint32_t>(G);
    }
    const int T = step_items(st, h);
    const int t0 = first_item(off);
    off = (off + static_cast<uint32_t>(T)) % static_cast<uint32_t>(G);
    if (t0 >= T) continue;  // no work for this CTA in this step
    ED_TRACE(p, s, 0, tid == 0 && t0 == 0);
    if (!is_umma_cell(st.cell)) {
      if (st.cell == ED_CELL_MVRNN_INTERNAL) {  // ---- MV-RNN matvecs: one CTA per item ----
        __syncthreads();  // sbias / swout are free (previous step's epilogue done)
        mv_vec_items<__nv_bfloat16>(p, st, t0, G, sbias, swout);
        if (tid == 0) stamp_step(p, s);
        continue;
      }
      // ---------------- SIMT step (output linear / tagger output): every warp, 2 rows each ----------
      const int C = st.gates;
      const bool in_smem = C * h * 4 <= kWoutBytes;
      if (p.has_split) __syncthreads();  // swout may still hold a split-K exchange of the epilogue
      if (in_smem) {  // 16 B cp.async per piece (no register staging)
        const float *W = static_cast<const float *>(step_W(p, st));
        const uint32_t sw = smem_u32(swout);
        for (int q = tid; q < C * h / 4; q += kThreadsTC) cp_async16(sw + 16u * q, W + 4 * q);
        cp_async_commit();
        cp_async_wait<0>();
      }
      __syncthreads();
      if (p.trace && tid == 0) p.trace[p.num_steps * 64 + blockIdx.x * 4 + 1] = globaltimer();
      const float *Ws = in_smem ? swout : static_cast<const float *>(step_W(p, st));
      for (int t = t0; t < T; t += G) linear_out_rows_bf16(p, st, static_cast<long>(t) * kSimtRows + 2 * warp, Ws);
      if (p.trace && lane == 0) atomicMax(p.trace + p.num_steps * 64 + blockIdx.x * 4 + 2, globaltimer());
      __syncthreads();  // swout is reused by the next SIMT step
      if (tid == 0) stamp_step(p, s);
      continue;
    }
    const int ncols = st.cell == ED_CELL_LINEAR_OUT ? 16 : st.gates * st.units;
    const int kc_total = (cell_segments_dev(st.cell) * h) / kChunkK;
    uint32_t abytes = kAStage;
    const int kc_part = split ? kc_total / 2 : kc_total;  // K chunks per CTA
    const int kps = step_kps(st, kc_part, &abytes);
    const uint32_t boff = kps > 1 ? kps * abytes : static_cast<uint32_t>(kAStage);  // B region of a stage
    const uint32_t bchunk = static_cast<uint32_t>(ncols) * 128u;
if (warp == 4) {
      // ---------------- MMA issuer ----------------
      for (int t = t0; t < T; t += G) {
        const uint32_t acc = pipe.ti & 1u;
        const int tile = split ? (t >> 1) : t;
        const int kbeg = split ? (t & 1) * kc_part : 0, kend = kbeg + kc_part;
        const uint32_t idesc = idesc_bf16(tile_cols(st, h, tile % st.n_col_tiles));
        // the whole warp walks the loop (warp-uniform operands); one elected lane issues
        mbar_wait_warp(tempty + acc, ((pipe.ti >> 1) & 1u) ^ 1u);
        tc_fence_after();
        const uint32_t d = tmem_base + acc * 256u;
        const uint64_t astep = abytes >> 4, bstep = bchunk >> 4;  // descriptor address units (16 B)
        for (int kc0 = kbeg; kc0 < kend; kc0 += kps) {
          const int nk = min(kps, kend - kc0);
          const uint32_t stg = pipe.it % kStages;
          mbar_wait_warp(full + stg, (pipe.it / kStages) & 1u);
          fence_proxy_async_smem();  // cp.async (generic proxy) rows -> tcgen05.mma (async proxy)
          tc_fence_after();
          ED_TRACE(p, s, 3, lane == 0 && kc0 == 0 && t == 0);
#ifdef ED_CHUNK_TRACE  // development: when each stage of item 0 became full (MMA side)
          ED_TRACE(p, s, 32 + min(15, (kc0 - kbeg) / kps), lane == 0 && t == 0);
#endif
          const uint32_t sbase = smem_u32(stages + stg * kStageBytes);
          uint64_t ad = sw128_desc(sbase), bd = sw128_desc(sbase + boff);
          for (int q = 0; q < nk; ++q, ad += astep, bd += bstep) {
#pragma unroll
            for (int k = 0; k < kChunkK / 16; ++k)
              tc_mma_elect(d, ad + 2 * k, bd + 2 * k, idesc, (kc0 + q > kbeg || k > 0) ? 1u : 0u);
          }
          tc_commit_elect(empty + stg);
          ++pipe.it;
        }
        tc_commit_elect(tfull + acc);
        ED_TRACE(p, s, 4, lane == 0 && t == 0);
        ++pipe.ti;
      }
    } else if (warp == 5) {
      // ---------------- weight (B) loader: runs ahead across steps (weights are static) -----------
      const uint8_t *Wp = static_cast<const uint8_t *>(step_W(p, st));
      const size_t ntot = st.cell == ED_CELL_LINEAR_OUT ? 16 : static_cast<size_t>(st.gates) * h;
      for (int t = t0; t < T; t += G) {  // warp-converged; one elected lane issues
        const int col_tile = (split ? (t >> 1) : t) % st.n_col_tiles;
        const int kbeg = split ? (t & 1) * kc_part : 0, kend = kbeg + kc_part;
        const uint32_t nb = static_cast<uint32_t>(tile_cols(st, h, col_tile)) * 128u;
        for (int kc0 = kbeg; kc0 < kend; kc0 += kps) {
          const int nk = min(kps, kend - kc0);
          const uint32_t stg = pipe.it % kStages;
          mbar_wait_warp(empty + stg, ((pipe.it / kStages) & 1u) ^ 1u);
#ifdef ED_CHUNK_TRACE  // development: when the weight loader got each stage of item 0
          ED_TRACE(p, s, 11 + min(15, (kc0 - kbeg) / kps), lane == 0 && t == 0);
#endif
          mbar_arrive_tx_elect(full + stg, nb * nk);
          for (int q = 0; q < nk; ++q) {
            const uint8_t *src =
                Wp + ((static_cast<size_t>(kc0 + q) * ntot + static_cast<size_t>(col_tile) * ncols) * 128);
            bulk_g2s_elect(stages + stg * kStageBytes + boff + q * bchunk, src, nb, full + stg);
          }
          ++pipe.it;
        }
      }
    } else {
      // ---------------- operand (A) loaders: warps 6-11 ----------------
      // Per tile: row table (static) -> wait until every input row is published (acquire) ->
      // CONTIG operand: one TMA 128-row box; gathered operand: 16 B cp.async per (row, chunk).
      // Every loader thread hands its part of a stage to the MMA with cp.async.mbarrier.arrive.noinc
      // (the stage completes when all gathered rows and TMA bytes have landed); the MMA thread fences
      // the generic -> async proxy before reading the stage.
      const int lt = tid - 192;  // 0 .. kLoaderThreads-1
      const int nseg = cell_segments_dev(st.cell);
      if (st.cell == kCellMvMat) {
        // MV-RNN matrix product: A rows = [A^T | B^T] rows of the children's matrices; each 64-row
        // half of a tile lies in one node's block -> two TMA boxes {64 cols, 64 rows} per stage,
        // from Mx (child node) or the packed word-matrix table (leaf).  No cp.async: stages are
        // released right after issue.
        const long mrows = static_cast<long>(st.m) * h;
        for (int t = t0; t < T; t += G) {
          const long R0 = static_cast<long>(t / st.n_col_tiles) * kTileM;
          int ent[2][2], rr0[2], nh = 0;
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const long R = R0 + q * 64;
            if (R < mrows) {
              const int node = static_cast<int>(R / h);
              rr0[q] = static_cast<int>(R % h);
              ent[q][0] = slot_entry(st, p.idx, 0, node);
              ent[q][1] = slot_entry(st, p.idx, 1, node);
              nh = q + 1;
            }
          }
          for (int q = 0; q < nh; ++q) {
            wait_row(p, ent[q][0], st);
            wait_row(p, ent[q][1], st);
          }
          asm volatile("fence.proxy.async.global;" ::: "memory");
          for (int kc = 0; kc < kc_total; ++kc) {
            const uint32_t stg = pipe.it % kStages;
            mbar_wait_warp(empty + stg, ((pipe.it / kStages) & 1u) ^ 1u);
            const int seg = (kc * kChunkK) / h, col0 = (kc * kChunkK) % h;
            uint8_t *a_dst = stages + stg * kStageBytes;
            if (lt == 0) {
              mbar_arrive_tx(full + stg, static_cast<uint32_t>(nh) * 8192u);
              for (int q = 0; q < nh; ++q) {
                const int e = ent[q][seg];
                if (e >= 0)
                  tma_row_box(a_dst + q * 8192, &p.tm_mx, col0, e * h + rr0[q], full + stg);
                else
                  tma_row_box(a_dst + q * 8192, &p.tm_mat[st.wset], col0, (-1 - e) * h + rr0[q], full + stg);
              }
            }
            cp_async_arrive_noinc(full + stg);
            ++pipe.it;
          }
        }
        continue;
      }
      for (int t = t0; t < T; t += G) {
        const int row_tile = (split ? (t >> 1) : t) / st.n_col_tiles;
        const int kbeg = split ? (t & 1) * kc_part : 0, kend = kbeg + kc_part;
        const void **tab = rowtab + (tab_tile & 1u) * (kTileM * 2);
        ++tab_tile;
        int ent[2][2];  // this thread's input rows (at most 2 rows x 2 segments)
        int nent = 0;
        for (int r = lt; r < kTileM; r += kLoaderThreads, ++nent) {
          const int i = row_tile * kTileM + r;
          const int iv = i < st.m ? i : (st.m - 1);  // rows past m repeat the last valid row
#pragma unroll
          for (int sg = 0; sg < 2; ++sg) {
            sts_ptr(tab + r * 2 + sg, sg < nseg ? static_cast<const void *>(segment_row<__nv_bfloat16>(p, st, sg, iv)) : p.H);
            ent[nent][sg] = sg < nseg ? segment_entry(p, st, sg, iv) : -1;
          }
        }
        // Readiness per K segment, just before its first chunk: the rows of segment sg are checked in
        // parallel (each thread its own rows, AND-reduced over the loader threads) and the threads
        // block only on the rows still pending.  A segment that is ready early (an LSTM's x, a leaf
        // child) is gathered and multiplied while the other segment's producers still run.
        auto acquire_seg = [&](int sg) {
          bool ok = true;
          for (int q = 0; q < nent; ++q) ok = ok && row_ready(p, ent[q][sg], st);
          int all_ok;
          asm volatile("{\n\t.reg .pred pi, po;\n\tsetp.ne.s32 pi, %1, 0;\n\t"
                       "bar.red.and.pred po, 1, %2, pi;\n\tselp.s32 %0, 1, 0, po;\n\t}"
                       : "=r"(all_ok) : "r"(static_cast<int>(ok)), "n"(kLoaderThreads) : "memory");
          if (!all_ok) {
            for (int q = 0; q < nent; ++q) wait_row(p, ent[q][sg], st);
            asm volatile("bar.sync 1, %0;" ::"n"(kLoaderThreads) : "memory");
          }
          asm volatile("fence.proxy.async.global;" ::: "memory");  // published rows may be read by TMA
        };
        const int sg0 = kbeg * kChunkK >= h ? 1 : 0;  // first K segment of this CTA's range
        acquire_seg(sg0);
        int acquired = sg0 + 1;  // segments [sg0, acquired) are acquired
        if (lt == 0) ED_TRACE(p, s, 1, t == 0);
        const int nrows = min(kTileM, st.m - row_tile * kTileM);
        const int pieces = nrows * 8;  // 16 B pieces per K chunk
        const float inv_pieces = 1.0f / static_cast<float>(pieces);
        int cb[2] = {-1, -1};  // per K segment: base row of its contiguous block, or -1 (gathered)
#pragma unroll
        for (int sg = 0; sg < 2; ++sg)
          if (sg < nseg && !segment_contig(p, st, sg, &cb[sg])) cb[sg] = -1;
        for (int kc0 = kbeg; kc0 < kend; kc0 += kps) {
          const int nk = min(kps, kend - kc0);
#ifdef ED_CHUNK_TRACE
          ED_TRACE(p, s, 27, lt == 0 && t == 0 && kc0 == kbeg + 4);
#endif
          if (acquired < 2 && (kc0 + nk - 1) * kChunkK >= h) {  // the stage reaches segment 1
            acquire_seg(1);
            acquired = 2;
          }
          const uint32_t stg = pipe.it % kStages;
          bool tma_stage = false;
#if ED_TMA_ROTATE >= 2
          // Stage ownership: loader warp (stage index) alone waits on a stage's empty barrier (so no
          // warp ever waits on a phase two uses ahead).  A stage read by one TMA box is handled by
          // its owner alone (one arrival of count 192 for the loader threads); a gathered stage is
          // released to all loader warps by a named barrier after the owner's wait.
          {
            const int sgq = (kc0 * kChunkK >= h) ? 1 : 0;
            const int cbq = (nk == 1 && kps == 1) ? (sgq ? cb[1] : cb[0]) : -1;
            const bool own = (lt >> 5) == static_cast<int>(stg);
            if (cbq >= 0) {
              if (own) {
                mbar_wait(empty + stg, ((pipe.it / kStages) & 1u) ^ 1u);
                uint8_t *a_dst = stages + stg * kStageBytes;
                const int col0q = kc0 * kChunkK - sgq * h;
                mbar_arrive_tx_elect(full + stg, kAStage);
                if (st.cell == kCellMvP)  // U rows: [B a | A b], 2h columns
                  tma_row_box_elect(a_dst, &p.tm_u, sgq * h + col0q, cbq + row_tile * kTileM, full + stg);
                else
                  tma_row_box_elect(a_dst, &p.tm_h128, col0q, cbq + row_tile * kTileM, full + stg);
                if ((lt & 31) == 0) mbar_arrive_cnt(full + stg, kLoaderThreads);
              }
              ++pipe.it;
              continue;
            }
            if (own) mbar_wait(empty + stg, ((pipe.it / kStages) & 1u) ^ 1u);
            asm volatile("bar.sync 3, %0;" ::"n"(kLoaderThreads) : "memory");
          }
#else
          mbar_wait_warp(empty + stg, ((pipe.it / kStages) & 1u) ^ 1u);
#endif
#ifdef ED_CHUNK_TRACE  // development: when the operand loaders got each stage of item 0
          ED_TRACE(p, s, 48 + min(15, (kc0 - kbeg) / kps), lt == 0 && t == 0);
#endif
          if (nk > 1) {  // several small chunks per stage: row gathers only (a 128-row box would overflow)
            if (lt == 0) mbar_arrive(full + stg);
            // the stage's nk x nrows x 8 pieces spread over all loader threads (a one-row tile puts
            // its nk chunks on 8 nk lanes at once instead of one chunk after another)
            const uint32_t a_base = smem_u32(stages + stg * kStageBytes);
            for (int c = lt; c < nk * pieces; c += kLoaderThreads) {
              const int q = static_cast<int>((static_cast<float>(c) + 0.5f) * inv_pieces);
              const int rem = c - q * pieces, r = rem >> 3, ch = rem & 7;
              const int kc = kc0 + q;
              const int seg = kc * kChunkK >= h ? 1 : 0, col0 = kc * kChunkK - seg * h;
              const __nv_bfloat16 *src = static_cast<const __nv_bfloat16 *>(lds_ptr(tab + r * 2 + seg)) + col0 + ch * 8;
              cp_async16(a_base + q * abytes + r * 128 + ((ch ^ (r & 7)) << 4), src);
            }
          } else {
          const int kc = kc0;
          const int seg = kc * kChunkK >= h ? 1 : 0, col0 = kc * kChunkK - seg * h;  // K = nseg * h, nseg <= 2
          uint8_t *a_dst = stages + stg * kStageBytes;
          // a 128-row box needs the full 16 KB A region: only with one chunk per stage (kps == 1)
          const int cbase = kps == 1 ? (seg == 0 ? cb[0] : cb[1]) : -1;
          tma_stage = cbase >= 0;
          if (cbase >= 0) {
            // the stage's TMA box is issued by loader warp (stage mod #loader warps): consecutive
            // chunks' issues run on different warps instead of one after another on warp 6
#if ED_TMA_ROTATE
            if ((lt >> 5) == static_cast<int>(stg % ED_LOADER_WARPS)) {
#else
            if (lt < 32) {  // warp-converged; one elected lane issues
#endif
              mbar_arrive_tx_elect(full + stg, kAStage);
              if (st.cell == kCellMvP)  // U rows: [B a | A b], 2h columns
                tma_row_box_elect(a_dst, &p.tm_u, seg * h + col0, cbase + row_tile * kTileM, full + stg);
              else
                tma_row_box_elect(a_dst, &p.tm_h128, col0, cbase + row_tile * kTileM, full + stg);
#ifdef ED_CHUNK_TRACE
              ED_TRACE(p, s, 28, lt == 0 && t == 0 && kc0 == kbeg + 4);
#endif
            }
          } else {
            if (lt == 0) mbar_arrive(full + stg);  // the TMA arrival slot is unused for this stage
            const uint32_t a_base = smem_u32(a_dst);
            for (int c = lt; c < nrows * 8; c += kLoaderThreads) {  // rows past m are not loaded
              const int r = c >> 3, ch = c & 7;
              const __nv_bfloat16 *src = static_cast<const __nv_bfloat16 *>(lds_ptr(tab + r * 2 + seg)) + col0 + ch * 8;
              cp_async16(a_base + r * 128 + ((ch ^ (r & 7)) << 4), src);
            }
          }
          }
          // the stage completes when this thread's gathers have landed (no software lag); a stage
          // read by TMA only takes one arrival standing for every loader thread (the per-thread
          // mbarrier arrivals are serialised by the barrier: ~0.45 us per stage for 192 threads)
#ifdef ED_CHUNK_TRACE
          ED_TRACE(p, s, 29, lt == 0 && t == 0 && kc0 == kbeg + 4);
#endif
#if ED_TMA_ONE_ARRIVE
          if (tma_stage) {
            if (lt == 0) mbar_arrive_cnt(full + stg, kLoaderThreads);
          } else {
            cp_async_arrive_noinc(full + stg);
          }
#else
          cp_async_arrive_noinc(full + stg);
#endif
#ifdef ED_CHUNK_TRACE
          ED_TRACE(p, s, 30, lt == 0 && t == 0 && kc0 == kbeg + 4);
#endif
          ++pipe.it;
        }
        if (lt == 0) ED_TRACE(p, s, 2, t == 0);
      }
    }
  }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 4) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
  if (p.has_split) cluster_sync_all();  // no CTA leaves while its partner may still address it
}

// ------------------------------------------------------------------------------------------------
// weight packing
// ------------------------------------------------------------------------------------------------
// bf16 tensor-core layout of a logical [G*h, K] matrix: [K/64][G*h][64] bf16, packed row p holds
// logical row g*h + j with p = (j/16)*(G*16) + g*16 + j%16 (gate-interleaved in 16-unit groups),
// and each 8-row x 128 B atom is 128B-swizzled (16 B chunk c of row r stored at c ^ (r & 7)).
__global__ void pack_umma_kernel(const float *src, __nv_bfloat16 *dst, int G, int h, int K, int valid_rows) {
  const long N = static_cast<long>(G) * h;
  const long total = N * K;
  for (long q = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; q < total;
       q += static_cast<long>(gridDim.x) * blockDim.x) {
    const long pr = q / K;       // packed row
    const int k = static_cast<int>(q % K);
    const long grp = pr / (G * 16);
    const int within = static_cast<int>(pr % (G * 16));
    const int g = within / 16;
    const long j = grp * 16 + within % 16;
    const long lr = static_cast<long>(g) * h + j;  // logical row (rows >= valid_rows are zero padding)
    const float v = lr < valid_rows ? src[lr * K + k] : 0.0f;
    const int kc = k / 64, kk = k % 64;
    const int ch = kk / 8, e = kk % 8;
    const long byte = (static_cast<long>(kc) * N + pr) * 128 + ((ch ^ static_cast<int>(pr & 7)) * 16) + e * 2;
    dst[byte / 2] = __float2bfloat16_rn(v);
  }
}

// SIMT layout: Wt[k][n] = W[n][k] (element type T).
template <typename T>
__global__ void pack_transpose_kernel(const float *src, T *dst, long N, long K) {
  const long total = N * K;
  for (long q = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; q < total;
       q += static_cast<long>(gridDim.x) * blockDim.x) {
    const long k = q / N, n = q % N;
    dst[q] = from_f<T>(src[n * K + k]);
  }
}

__global__ void copy_f32_kernel(const float *src, float *dst, long n) {
  for (long q = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; q < n;
       q += static_cast<long>(gridDim.x) * blockDim.x)
    dst[q] = src[q];
}

static bool umma_cell_host(int cell) {
  return cell == ED_CELL_TREELSTM_LEAF || cell == ED_CELL_TREELSTM_INTERNAL || cell == ED_CELL_TREEGRU_LEAF ||
         cell == ED_CELL_TREEGRU_INTERNAL || cell == ED_CELL_TREEFC_INTERNAL || cell == ED_CELL_LSTM ||
         cell == ED_CELL_LATTICE_CHAR || cell == ED_CELL_LATTICE_WORD || cell == ED_CELL_TAGGER ||
         cell == ED_CELL_LATTICEGRU_CHAR || cell == ED_CELL_LATTICEGRU_WORD ||
         cell == ED_CELL_MVRNN_INTERNAL;
}

// MV-RNN word-matrix table: dst[w][k][i] = src[w][i][k] (each matrix transposed), element type T.
template <typename T>
__global__ void pack_mat_transpose_kernel(const float *src, T *dst, long words, int h) {
  const long hh = static_cast<long>(h) * h;
  const long total = words * hh;
  for (long q = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; q < total;
       q += static_cast<long>(gridDim.x) * blockDim.x) {
    const long w = q / hh;
    const int k = static_cast<int>((q % hh) / h), i = static_cast<int>(q % h);
    dst[q] = from_f<T>(src[w * hh + static_cast<long>(i) * h + k]);
  }
}

// Logical shape of a cell's matrices (rows, cols).
static void logical_shape(int cell, int h, int out_dim, int which, long *rows, long *cols) {
  if (cell == ED_CELL_LINEAR_OUT) { *rows = out_dim; *cols = h; return; }
  if (which == 2) {  // MV-RNN word-matrix table [out_dim words][h][h]
    if (cell != ED_CELL_MVRNN_INTERNAL) { *rows = 0; *cols = 0; return; }
    *rows = static_cast<long>(out_dim) * h; *cols = h; return;
  }
  if (which == 1) {
    if (cell == ED_CELL_TAGGER) { *rows = out_dim; *cols = h; return; }
    *rows = h; *cols = 2 * h; return;   // lattice link gate W_l, MV-RNN W_M
  }
  *rows = static_cast<long>(cell_gates(cell)) * h;
  *cols = static_cast<long>(cell_segments(cell)) * h;
}

int64_t packed_bytes(int cell, int hidden, int out_dim, int dtype, int which) {
  long rows = 0, cols = 0;
  logical_shape(cell, hidden, out_dim, which, &rows, &cols);
  if (cell == ED_CELL_LINEAR_OUT && dtype == ED_BF16) return 16 * cols * 2;  // UMMA layout, N = 16 (zero rows >= C)
  if (cell == ED_CELL_LINEAR_OUT || (cell == ED_CELL_TAGGER && which == 1)) return rows * cols * 4;
  return rows * cols * (dtype == ED_BF16 ? 2 : 4);
}

int launch_pack(int cell, int hidden, int out_dim, int dtype, int which, const float *src, void *dst,
                void *stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  long rows = 0, cols = 0;
  logical_shape(cell, hidden, out_dim, which, &rows, &cols);
  const int threads = 256;
  const long total = rows * cols;
  const int blocks = static_cast<int>((total + threads - 1) / threads < 4096 ? (total + threads - 1) / threads : 4096);
  if (total == 0) return which == 2 && cell != ED_CELL_MVRNN_INTERNAL ? static_cast<int>(cudaErrorInvalidValue) : 0;
  if (which == 2) {
    if (dtype == ED_BF16)
      pack_mat_transpose_kernel<__nv_bfloat16><<<blocks, threads, 0, s>>>(src, static_cast<__nv_bfloat16 *>(dst), out_dim, hidden);
    else
      pack_mat_transpose_kernel<float><<<blocks, threads, 0, s>>>(src, static_cast<float *>(dst), out_dim, hidden);
  } else if (cell == ED_CELL_LINEAR_OUT && dtype == ED_BF16) {
    if (hidden % 64 != 0) return static_cast<int>(cudaErrorInvalidValue);
    const long total16 = 16 * cols;
    const int b16 = static_cast<int>((total16 + threads - 1) / threads);
    pack_umma_kernel<<<b16, threads, 0, s>>>(src, static_cast<__nv_bfloat16 *>(dst), 1, 16, static_cast<int>(cols),
                                             static_cast<int>(rows));
  } else if (cell == ED_CELL_LINEAR_OUT || (cell == ED_CELL_TAGGER && which == 1)) {
    copy_f32_kernel<<<blocks, threads, 0, s>>>(src, static_cast<float *>(dst), total);
  } else if (dtype == ED_BF16 && umma_cell_host(cell) &&
             (which == 0 || cell == ED_CELL_LATTICE_WORD || cell == ED_CELL_MVRNN_INTERNAL)) {
    if (hidden % 64 != 0) return static_cast<int>(cudaErrorInvalidValue);
    const int G = which == 0 ? cell_gates(cell) : 1;  // link gate W_l: one gate block
    pack_umma_kernel<<<blocks, threads, 0, s>>>(src, static_cast<__nv_bfloat16 *>(dst), G, hidden,
                                                static_cast<int>(cols), static_cast<int>(rows));
  } else if (dtype == ED_BF16) {
    pack_transpose_kernel<__nv_bfloat16><<<blocks, threads, 0, s>>>(src, static_cast<__nv_bfloat16 *>(dst), rows, cols);
  } else {
    pack_transpose_kernel<float><<<blocks, threads, 0, s>>>(src, static_cast<float *>(dst), rows, cols);
  }
  return static_cast<int>(cudaGetLastError());
}

// ------------------------------------------------------------------------------------------------
// launch
// ------------------------------------------------------------------------------------------------
static int device_query(int dev, int *sm_count, int *major, int *minor);
int device_check(int *sm_count, int *major, int *minor) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return static_cast<int>(e);
  // device attributes do not change: queried once per device
  constexpr int kMaxDev = 64;
  static std::mutex mu;
  static int known[kMaxDev][4] = {};
  if (dev >= 0 && dev < kMaxDev) {
    std::lock_guard<std::mutex> lk(mu);
    if (known[dev][0]) {
      *sm_count = known[dev][1];
      *major = known[dev][2];
      *minor = known[dev][3];
      return 0;
    }
  }
  const int r = device_query(dev, sm_count, major, minor);
  if (r == 0 && dev >= 0 && dev < kMaxDev) {
    std::lock_guard<std::mutex> lk(mu);
    known[dev][1] = *sm_count;
    known[dev][2] = *major;
    known[dev][3] = *minor;
    known[dev][0] = 1;
  }
  return r;
}

static int device_query(int dev, int *sm_count, int *major, int *minor) {
  cudaError_t e;
  e = cudaDeviceGetAttribute(sm_count, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return static_cast<int>(e);
  e = cudaDeviceGetAttribute(major, cudaDevAttrComputeCapabilityMajor, dev);
  if (e != cudaSuccess) return static_cast<int>(e);
  e = cudaDeviceGetAttribute(minor, cudaDevAttrComputeCapabilityMinor, dev);
  return static_cast<int>(e);
}

// Launch configuration of a plan with split-K steps: clusters of 2 CTAs (one per SM).
static void cluster2_config(cudaLaunchConfig_t *cfg, cudaLaunchAttribute *at, int grid, cudaStream_t s,
                            bool cooperative) {
  std::memset(cfg, 0, sizeof(*cfg));
  cfg->gridDim = dim3(grid);
  cfg->blockDim = dim3(kThreadsTC);
  cfg->dynamicSmemBytes = kSmemBytes;
  cfg->stream = s;
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeCooperative;
  at[1].val.cooperative = 1;
  cfg->attrs = at;
  cfg->numAttrs = cooperative ? 2 : 1;
}

static int persistent_grid_uncached(int dtype, bool cluster2, int *grid);
// The occupancy queries cost tens of us per call: one result per (device, dtype, cluster launch),
// so a serving loop's new minibatch plans do not pay them on every first execute.
static int persistent_grid_cached(int dtype, bool cluster2, int *grid);
// ED_GRID_MAX (testing): cap the persistent grid (rounded down to even for cluster launches), so
// that batches get several tiles per CTA (split-K pairs exchange more than once per batch).
int persistent_grid(int dtype, bool cluster2, int *grid) {
  const int e = persistent_grid_cached(dtype, cluster2, grid);
  const char *cap = std::getenv("ED_GRID_MAX");
  if (e == 0 && cap && std::atoi(cap) > 0 && *grid > std::atoi(cap)) {
    *grid = std::atoi(cap);
    if (cluster2) *grid &= ~1;
    if (*grid < 2) *grid = 2;
  }
  return e;
}

static int persistent_grid_cached(int dtype, bool cluster2, int *grid) {
  constexpr int kMaxDev = 64;
  static std::mutex mu;
  static int cache[kMaxDev][2][2] = {};
  int dev = 0;
  cudaError_t ce = cudaGetDevice(&dev);
  if (ce != cudaSuccess) return static_cast<int>(ce);
  const int d = dtype == ED_BF16 ? 1 : 0, c = cluster2 ? 1 : 0;
  if (dev >= 0 && dev < kMaxDev) {
    std::lock_guard<std::mutex> lk(mu);
    if (cache[dev][d][c] > 0) {
      *grid = cache[dev][d][c];
      return 0;
    }
  }
  const int e = persistent_grid_uncached(dtype, cluster2, grid);
  if (e == 0 && dev >= 0 && dev < kMaxDev) {
    std::lock_guard<std::mutex> lk(mu);
    cache[dev][d][c] = *grid;
  }
  return e;
}

static int persistent_grid_uncached(int dtype, bool cluster2, int *grid) {
  int sms = 0, major = 0, minor = 0;
  int e = device_check(&sms, &major, &minor);
  if (e) return e;
  int per_sm = 0;
  if (dtype == ED_BF16) {
    cudaError_t ce = cudaFuncSetAttribute(ed_persistent_bf16, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    if (ce != cudaSuccess) return static_cast<int>(ce);
    ce = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ed_persistent_bf16, kThreadsTC, kSmemBytes);
    if (ce != cudaSuccess) return static_cast<int>(ce);
    if (per_sm > 1) per_sm = 1;  // TMEM: one 512-column allocation per SM
    if (cluster2) {
      // every CTA must be resident at once (dataflow waits): as many pairs as fit together
      cudaLaunchConfig_t cfg;
      cudaLaunchAttribute at[2];
      cluster2_config(&cfg, at, 2 * (sms / 2), nullptr, false);
      int clusters = 0;
      ce = cudaOccupancyMaxActiveClusters(&clusters, ed_persistent_bf16, &cfg);
      if (ce != cudaSuccess) return static_cast<int>(ce);
      *grid = 2 * (clusters < sms / 2 ? clusters : sms / 2);
      return *grid > 0 ? 0 : static_cast<int>(cudaErrorLaunchOutOfResources);
    }
  } else {
    cudaError_t ce = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ed_persistent_f32, kThreads, 0);
    if (ce != cudaSuccess) return static_cast<int>(ce);
    if (per_sm > 2) per_sm = 2;
  }
  *grid = sms * (per_sm > 0 ? per_sm : 1);
  return 0;
}

int launch_persistent(const KParams &p, int dtype, int grid, bool cluster2, void *stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  void *args[] = {const_cast<KParams *>(&p)};
  if (dtype == ED_BF16 && cluster2) {
    cudaLaunchConfig_t cfg;
    cudaLaunchAttribute at[2];
    // Not a cooperative launch: ncu cannot replay cooperative cluster launches (LaunchFailed), and
    // the grid is sized by cudaOccupancyMaxActiveClusters so that every pair is resident at once on
    // an idle GPU (the dataflow waits need that).  ED_CLUSTER_COOP=1 asks for the cooperative form.
    static const bool coop = std::getenv("ED_CLUSTER_COOP") && std::atoi(std::getenv("ED_CLUSTER_COOP")) == 1;
    cluster2_config(&cfg, at, grid, s, coop);
    e = cudaLaunchKernelExC(&cfg, reinterpret_cast<const void *>(ed_persistent_bf16), args);
    if (e == cudaErrorInvalidValue || e == cudaErrorNotSupported) {  // cooperative + cluster not accepted:
      (void)cudaGetLastError();                                       // the grid is sized to be co-resident
      cluster2_config(&cfg, at, grid, s, false);
      e = cudaLaunchKernelExC(&cfg, reinterpret_cast<const void *>(ed_persistent_bf16), args);
    }
  } else if (dtype == ED_BF16) {
    e = cudaLaunchCooperativeKernel(reinterpret_cast<void *>(ed_persistent_bf16), dim3(grid), dim3(kThreadsTC), args,
                                    kSmemBytes, s);
  } else {
    e = cudaLaunchCooperativeKernel(reinterpret_cast<void *>(ed_persistent_f32), dim3(grid), dim3(kThreads), args, 0,
                                    s);
  }
  return static_cast<int>(e);
}

}  // namespace ed
