// Probe: the persistent kernel's K-loop pipeline in isolation (sm_100a, 148 CTAs x 384 threads).
// Per item: KC stages, each = A tile (128 rows x 64 bf16: one TMA box, or 16 B cp.async row gathers
// by 192 loader threads) + B tile (N rows x 128 B, one cp.async.bulk) -> 4 x tcgen05.mma M=128 K=16.
// Ring of S stages (full/empty mbarriers), 2 TMEM accumulators handed to 4 epilogue warps.
// Reports ns per stage (mean over CTAs).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/ring_probe scripts/ring_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cstdlib>

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t *b, uint32_t par) {
  uint32_t ok = 0, n = 0;
  while (!ok) {
    if (++n > (1u << 22)) __trap();
    asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                 : "=r"(ok) : "r"(sa(b)), "r"(par) : "memory");
  }
}
__device__ __forceinline__ uint64_t desc(uint32_t saddr) {
  return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__device__ __forceinline__ uint32_t idesc(int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

struct Cfg {
  int S, N, KC, items, amode, mma, rows, tiles, kps;
};

__global__ void __launch_bounds__(384, 1) probe(const __grid_constant__ CUtensorMap mh, const __grid_constant__ CUtensorMap mh3,
                                                const __grid_constant__ CUtensorMap mw3, const uint8_t *H,
                                                const uint8_t *W, Cfg c, unsigned long long *out) {
  extern __shared__ uint8_t smraw[];
  uint8_t *sm = (uint8_t *)(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
  const int stage_bytes = c.kps * (16384 + ((c.N * 128 + 1023) & ~1023));
  const int boff = c.kps * 16384;
  uint64_t *full = (uint64_t *)(sm + c.S * stage_bytes);
  uint64_t *empty = full + 8, *tfull = full + 16, *tempty = full + 18;
  uint32_t *tslot = (uint32_t *)(full + 24);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nload = c.amode == 1 ? 192 : 1;
  if (tid == 0) {
    for (int s = 0; s < c.S; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(full + s)), "r"(1 + nload));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(empty + s)));
    }
    for (int a = 0; a < 2; ++a) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(tfull + a)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 128;" ::"r"(sa(tempty + a)));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 4) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(sa(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tbase = *tslot;
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  const int total = c.items * c.KC / c.kps;
  if (warp == 4) {
    for (int it = 0, ti = 0; ti < c.items; ++ti) {
      const uint32_t acc = ti & 1;
      wait(tempty + acc, ((ti >> 1) & 1) ^ 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      for (int kc = 0; kc < c.KC; kc += c.kps, ++it) {
        const int s = it % c.S;
        wait(full + s, (it / c.S) & 1);
        if (blockIdx.x == 0 && lane == 0 && it < 64) { unsigned long long tt; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt)); out[4096 + it] = tt - t0; }
        if (c.mma != 2) asm volatile("fence.proxy.async.shared::cta;");
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t base = sa(sm + s * stage_bytes);
        if (c.mma) {
          for (int k = 0; k < 4 * c.kps; ++k) {
            uint64_t ad = desc(base + (k >> 2) * 16384) + 2 * (k & 3), bd = desc(base + boff + (k >> 2) * c.N * 128) + 2 * (k & 3);
            uint32_t accf = (kc > 0 || k > 0);
            asm volatile(
                "{.reg .pred p, e; elect.sync _|e, 0xffffffff; setp.ne.b32 p, %4, 0;\n\t"
                "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}" ::"r"(tbase + acc * 256),
                "l"(ad), "l"(bd), "r"(idesc(c.N)), "r"(accf)
                : "memory");
          }
          asm volatile(
              "{.reg .pred e; elect.sync _|e, 0xffffffff;\n\t"
              "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];}" ::"r"(sa(empty + s))
              : "memory");
        } else if (lane == 0) {
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(empty + s)) : "memory");
        }
      }
      if (c.mma)
        asm volatile(
            "{.reg .pred e; elect.sync _|e, 0xffffffff;\n\t"
            "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];}" ::"r"(sa(tfull + acc))
            : "memory");
      else if (lane == 0)
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(tfull + acc)) : "memory");
    }
  } else if (warp == 5) {
    const int col_tile = blockIdx.x % c.tiles;
    for (int it = 0; it < total; ++it) {
      const int s = it % c.S, kc = (it * c.kps) % c.KC;
      wait(empty + s, ((it / c.S) & 1) ^ 1);
      if (lane == 0 && c.amode == 3) {
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(full + s)) : "memory");
      } else if (lane == 0 && c.amode == 4) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(full + s)), "r"(c.N * 128 * c.kps) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
                sa(sm + s * stage_bytes + boff)),
            "l"(&mw3), "r"(0), "r"(col_tile * c.N), "r"(kc), "r"(sa(full + s))
            : "memory");
      } else if (lane == 0) {
        const uint32_t nb = c.N * 128;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(full + s)), "r"(nb * c.kps) : "memory");
        for (int q = 0; q < c.kps; ++q) {
        const uint8_t *src = W + ((size_t)(kc + q) * c.tiles * c.N + (size_t)col_tile * c.N) * 128;
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                sa(sm + s * stage_bytes + boff + q * nb)),
            "l"(src), "r"(nb), "r"(sa(full + s))
            : "memory");
        }
      }
    }
  } else if (warp >= 6) {
    const int lt = tid - 192;
    for (int it = 0; it < total; ++it) {
      const int s = it % c.S, kc = (it * c.kps) % c.KC, item = (it * c.kps) / c.KC;
      const int row0 = (int)(((unsigned)(blockIdx.x * 7 + item * 13) * 128u) % (unsigned)(c.rows - 128));
      if (c.amode == 6 && (lt >> 5) != it % 6) continue;
      wait(empty + s, ((it / c.S) & 1) ^ 1);
      if (blockIdx.x == 0 && (lt & 31) == 0 && it < 64) { unsigned long long tt; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt)); out[2048 + it] = tt - t0; }
      if (c.amode == 4) {
        if (lt == 0) {
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(full + s)), "r"(16384 * c.kps) : "memory");
          asm volatile(
              "cp.async.bulk.tensor.3d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
                  sa(sm + s * stage_bytes)),
              "l"(&mh3), "r"(0), "r"(row0), "r"(kc % 8), "r"(sa(full + s))
              : "memory");
        }
      } else if (c.amode == 2) {  // kps separate 2-D boxes
        if (lt == 0) {
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(full + s)), "r"(16384 * c.kps) : "memory");
          for (int q = 0; q < c.kps; ++q)
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                    sa(sm + s * stage_bytes + q * 16384)),
                "l"(&mh), "r"(((kc + q) % 8) * 64), "r"(row0), "r"(sa(full + s))
                : "memory");
        }
      } else if (c.amode == 5) {
        if (lt == 0) {
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(full + s)), "r"(16384 * c.kps) : "memory");
          const uint8_t *src = H + (size_t)row0 * 1024 + (size_t)(kc % 8) * 16384 * 0;
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  sa(sm + s * stage_bytes)),
              "l"(src), "r"(16384 * c.kps), "r"(sa(full + s))
              : "memory");
        }
      } else if (c.amode == 6) {  // rotate the issuing warp per stage
        if (lt == (it % 6) * 32) {
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(full + s)), "r"(16384) : "memory");
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                  sa(sm + s * stage_bytes)),
              "l"(&mh), "r"((kc % 8) * 64), "r"(row0), "r"(sa(full + s))
              : "memory");
        }
      } else if (c.amode == 0 || c.amode == 3) {
        if (lt == 0) {
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(full + s)), "r"(16384) : "memory");
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                  sa(sm + s * stage_bytes)),
              "l"(&mh), "r"((kc % 8) * 64), "r"(row0), "r"(sa(full + s))
              : "memory");
        }
      } else {
        const uint32_t abase = sa(sm + s * stage_bytes);
        for (int q = lt; q < 1024; q += 192) {
          const int r = q >> 3, ch = q & 7;
          // pseudo-random row (gather)
          const int gr = (int)(((unsigned)(row0 + r) * 2654435761u) % (unsigned)c.rows);
          const uint8_t *src = H + (size_t)gr * 1024 + (kc % 8) * 128 + ch * 16;
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(abase + r * 128 + ((ch ^ (r & 7)) << 4)),
                       "l"(src)
                       : "memory");
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(sa(full + s)) : "memory");
      }
    }
  } else {  // epilogue warps: wait for the accumulator, read 16 columns, free it
    for (int ti = 0; ti < c.items; ++ti) {
      const uint32_t acc = ti & 1;
      wait(tfull + acc, (ti >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      uint32_t r[8];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                   : "r"(tbase + ((uint32_t)(warp * 32) << 16) + acc * 256));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (r[0] == 0x7fffffff) out[1024 + tid] = r[1];
      asm volatile("tcgen05.fence::before_thread_sync;");
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(tempty + acc)) : "memory");
    }
  }
  unsigned long long t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 4) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
  if (tid == 128) out[blockIdx.x] = t1 - t0;  // MMA warp's last lane? use epilogue end time
}

typedef CUresult (*EncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                             const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char **argv) {
  setvbuf(stdout, nullptr, _IONBF, 0);
  const int only = argc > 1 ? atoi(argv[1]) : -1;
  int vi = -1;
  const int rows = 24000, h = 512;
  uint8_t *H, *W;
  unsigned long long *dout;
  cudaMalloc(&H, (size_t)rows * h * 2);
  cudaMemset(H, 0, (size_t)rows * h * 2);
  cudaMalloc(&W, (size_t)16 * 2560 * 128);
  cudaMemset(W, 0, (size_t)16 * 2560 * 128);
  cudaMalloc(&dout, 4096 * 8);
  EncodeFn enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q);
  CUtensorMap mh;
  cuuint64_t dims[2] = {(cuuint64_t)h, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)h * 2};
  cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
  enc(&mh, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, H, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUtensorMap mh3, mw3, mh64;
  (void)mh64;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  struct V { int S, N, amode, mma; const char *name; int kps; } vs[] = {
      {4, 80, 3, 1, "S4 N80 A-only mma"}, {4, 80, 2, 1, "S4 N80 2xA mma"}, {4, 80, 4, 1, "S4 N80 3D-kps2 mma"},
      {4, 80, 4, 0, "S4 N80 3D-kps2 nomma"}, {3, 240, 4, 1, "S3 N240 3D-kps2 mma"},
      {4, 80, 0, 1, "S4 N80 TMA mma"},   {7, 80, 0, 1, "S7 N80 TMA mma"},  {4, 80, 0, 0, "S4 N80 TMA nomma"},
      {4, 240, 0, 1, "S4 N240 TMA mma"}, {4, 80, 1, 1, "S4 N80 gather mma"}, {7, 80, 1, 1, "S7 N80 gather mma"},
      {2, 80, 0, 1, "S2 N80 TMA mma"},   {8, 80, 0, 1, "S8 N80 TMA mma"}, {4, 160, 0, 1, "S4 N160 TMA mma"},
      {4, 80, 5, 1, "S4 N80 bulkA k1 mma", 1}, {4, 80, 5, 1, "S4 N80 bulkA k2 mma", 2}, {2, 80, 5, 1, "S2 N80 bulkA k4 mma", 4},
      {6, 80, 5, 1, "S6 N80 bulkA k1 mma", 1}, {4, 80, 5, 0, "S4 N80 bulkA k1 nomma", 1}, {2, 80, 4, 1, "S2 N80 3D-kps4 mma", 4},
      {4, 240, 5, 1, "S4 N240 bulkA k1 mma", 1},
      {2, 80, 2, 1, "S2 N80 4x2D k4 mma", 4}, {4, 80, 2, 1, "S4 N80 2x2D k2 mma", 2}, {2, 80, 4, 1, "S2 N80 3D k3 mma", 3},
      {2, 240, 2, 1, "S2 N240 2x2D k2 mma", 2}, {2, 240, 4, 1, "S2 N240 3D k2 mma", 2}, {3, 80, 2, 1, "S3 N80 2x2D k2 mma", 2},
      {4, 80, 0, 2, "S4 N80 TMA mma nofence", 1}, {4, 80, 2, 2, "S4 N80 2x2D k2 mma nofence", 2}, {4, 240, 0, 2, "S4 N240 TMA mma nofence", 1},
      {2, 80, 4, 2, "S2 N80 3D k4 mma nofence", 4},
      {4, 80, 6, 1, "S4 N80 TMA rot6 mma", 1}, {6, 80, 6, 1, "S6 N80 TMA rot6 mma", 1}, {4, 240, 6, 1, "S4 N240 TMA rot6 mma", 1}};
  for (auto &v : vs) {
    if (only >= 0 && ++vi != only) continue;
    printf("running %s\n", v.name);
    const int kps = v.kps ? v.kps : (v.amode == 4 ? 2 : 1);
    Cfg c{v.S, v.N, 16, 8, v.amode, v.mma, rows, 2560 / v.N, kps};
  {
    cuuint64_t d3[3] = {64, (cuuint64_t)rows, (cuuint64_t)(h / 64)};
    cuuint64_t s3[2] = {(cuuint64_t)h * 2, 128};
    cuuint32_t b3[3] = {64, 128, (cuuint32_t)kps}, e3[3] = {1, 1, 1};
    CUresult r = enc(&mh3, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, H, d3, s3, b3, e3, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r) printf("mh3 encode failed %d\n", (int)r);
  }
    {
      cuuint64_t d3[3] = {64, 2560, 16};
      cuuint64_t s3[2] = {128, 2560 * 128};
      cuuint32_t b3[3] = {64, (cuuint32_t)v.N, (cuuint32_t)kps}, e3[3] = {1, 1, 1};
      CUresult r = enc(&mw3, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, W, d3, s3, b3, e3, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r) printf("mw3 encode failed %d\n", (int)r);
    }
    const int stage_bytes = kps * (16384 + ((v.N * 128 + 1023) & ~1023));
    const int smem = 1024 + v.S * stage_bytes + 256;
    if (smem > 227 * 1024) { printf("%s: smem too big\n", v.name); continue; }
    for (int grid : {148, 64}) {
      for (int rep = 0; rep < 3; ++rep) probe<<<grid, 384, smem>>>(mh, mh3, mw3, H, W, c, dout);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("%s: %s\n", v.name, cudaGetErrorString(e)); return 1; }
      std::vector<unsigned long long> t(grid);
      cudaMemcpy(t.data(), dout, grid * 8, cudaMemcpyDeviceToHost);
      double avg = 0;
      for (auto x : t) avg += x;
      avg /= grid;
      const double per = avg / (c.items * c.KC / kps);
      printf("%-22s grid %3d: %6.0f ns/stage, %6.1f GB/s per SM (A+B)\n", v.name, grid, per,
             kps * (16384.0 + v.N * 128) / per);
      if (grid == 148) {
        std::vector<unsigned long long> ta(64), tf(64);
        cudaMemcpy(ta.data(), dout + 2048, 64 * 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(tf.data(), dout + 4096, 64 * 8, cudaMemcpyDeviceToHost);
        printf("  A free: "); for (int i = 0; i < 24; ++i) printf("%llu ", ta[i]); printf("\n");
        printf("  full:   "); for (int i = 0; i < 24; ++i) printf("%llu ", tf[i]); printf("\n");
      }
    }
  }
  return 0;
}
