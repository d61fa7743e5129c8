// Probe: does an SM overlap several TMA loads?  One thread issues NB loads of 16 KB (128 rows x 128 B,
// 128B swizzle) into NB distinct smem buffers, one mbarrier each, then waits for all of them.
// Modes: 0 = 2-D tile box {64, 128}; 1 = cp.async.bulk of 16 KB contiguous; 2 = 32 x tile::gather4
// (4 rows each, scattered rows); 3 = 16 B cp.async by 128 threads (scattered rows).
// Source: a 24 MB bf16 [24000 x 512] tensor (L2-resident after the first pass).  Reports ns for NB loads
// (median over CTAs, 3rd repetition), grid 1 and 148.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/tma_inflight_probe.bin scripts/tma_inflight_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t gt() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(128, 1) probe(const __grid_constant__ CUtensorMap m, const uint8_t *H, int mode, int nb,
                                                int rep_seed, unsigned long long *out) {
  extern __shared__ uint8_t smraw[];
  uint8_t *sm = (uint8_t *)(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
  uint64_t *bar = (uint64_t *)(sm + 12 * 16384);
  if (threadIdx.x == 0) {
    for (int b = 0; b < nb; ++b)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(bar + b)), "r"(mode == 3 ? 128 : 1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const unsigned base_row = (blockIdx.x * 977u + rep_seed * 131u) % 20000u;
  const uint64_t t0 = gt();
  if (mode == 3) {
    for (int b = 0; b < nb; ++b) {
      const uint32_t dst = sa(sm + b * 16384);
      for (int q = threadIdx.x; q < 1024; q += 128) {
        const int r = q >> 3, ch = q & 7;
        const unsigned gr = (base_row + r * 37u + b * 1009u) % 24000u;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + r * 128 + ((ch ^ (r & 7)) << 4)),
                     "l"(H + (size_t)gr * 1024 + (b & 7) * 128 + ch * 16)
                     : "memory");
      }
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(sa(bar + b)) : "memory");
    }
  } else if (threadIdx.x == 0) {
    for (int b = 0; b < nb; ++b) {
      const uint32_t dst = sa(sm + b * 16384);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(bar + b)), "r"(16384) : "memory");
      const int row = (int)((base_row + b * 1009u) % 23800u);
      if (mode == 0) {
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
            "l"(&m), "r"((b & 7) * 64), "r"(row), "r"(sa(bar + b))
            : "memory");
      } else if (mode == 1) {
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                     "l"(H + (size_t)row * 1024), "r"(16384), "r"(sa(bar + b))
                     : "memory");
      } else {
        for (int g = 0; g < 32; ++g) {
          int r[4];
          for (int k = 0; k < 4; ++k) r[k] = (int)((base_row + (4 * g + k) * 37u + b * 1009u) % 24000u);
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
              "%5, %6}], [%7];" ::"r"(dst + g * 512),
              "l"(&m), "r"((b & 7) * 64), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(sa(bar + b))
              : "memory");
        }
      }
    }
  }
  for (int b = 0; b < nb; ++b) {
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p;}"
                   : "=r"(ok) : "r"(sa(bar + b)) : "memory");
  }
  const uint64_t t1 = gt();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

typedef CUresult (*EncFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *, const cuuint64_t *,
                          const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int rows = 24000, h = 512;
  uint8_t *H;
  cudaMalloc(&H, (size_t)rows * h * 2);
  cudaMemset(H, 0, (size_t)rows * h * 2);
  unsigned long long *dout;
  cudaMalloc(&dout, 148 * 8);
  EncFn enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q);
  CUtensorMap m, m4;
  cuuint64_t d[2] = {(cuuint64_t)h, (cuuint64_t)rows};
  cuuint64_t s[1] = {(cuuint64_t)h * 2};
  cuuint32_t b[2] = {64, 128}, e[2] = {1, 1};
  enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, H, d, s, b, e, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cuuint32_t b4[2] = {64, 1};
  enc(&m4, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, H, d, s, b4, e, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int smem = 12 * 16384 + 1024 + 256;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char *names[] = {"tile box 16KB", "bulk 16KB", "gather4 x32", "cp.async 16B x1024"};
  for (int mode = 0; mode < 4; ++mode)
    for (int grid : {1, 148})
      for (int nb : {1, 2, 4, 8, 12}) {
        std::vector<unsigned long long> t(grid);
        for (int rep = 0; rep < 3; ++rep) probe<<<grid, 128, smem>>>(mode == 2 ? m4 : m, H, mode, nb, rep, dout);
        cudaError_t err = cudaDeviceSynchronize();
        if (err != cudaSuccess) { printf("mode %d: %s\n", mode, cudaGetErrorString(err)); return 1; }
        cudaMemcpy(t.data(), dout, grid * 8, cudaMemcpyDeviceToHost);
        std::sort(t.begin(), t.end());
        const double med = (double)t[grid / 2];
        printf("%-20s grid %3d nb %2d: %7.0f ns  (%6.1f GB/s per SM, %5.0f ns per load)\n", names[mode], grid, nb, med,
               nb * 16384.0 / med, med / nb);
      }
  return 0;
}
