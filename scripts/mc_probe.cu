// Probe: TMA tile::gather4 with .multicast::cluster inside clusters of CS CTAs (sm_100a).
// Every stage = 128 random rows x 128 B delivered to every CTA of the cluster; each CTA issues
// 32/CS gather4 ops with ctaMask = all CTAs.  Consumers free a stage cluster-wide (each CTA arrives
// on every CTA's empty barrier through mapa/remote arrive).  Reports per-stage time.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/mc_probe scripts/mc_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint32_t b, uint32_t par) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                 : "=r"(ok) : "r"(b), "r"(par) : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_n() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}

__global__ void probe(const __grid_constant__ CUtensorMap m1, int rows, int stages, int iters, int mc,
                      unsigned long long *out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t *buf = (uint8_t *)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  uint64_t *full = (uint64_t *)(buf + stages * 16384);
  uint64_t *empty = full + stages;
  const int lane = threadIdx.x;
  const uint32_t cr = cluster_rank(), cn = cluster_n();
  if (lane == 0) {
    for (int s = 0; s < stages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(full + s)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(empty + s)), "r"(cn));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  const int per = 32 / (mc ? cn : 1);  // gather4 ops per CTA per stage
  const uint16_t mask = (uint16_t)((1u << cn) - 1);
  auto issue = [&](int it) {
    const int s = it % stages;
    const uint32_t ph = (it / stages) & 1;
    wait(sa(empty + s), ph ^ 1);  // every CTA of the cluster freed this stage
    if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(full + s)), "r"(16384) : "memory");
    __syncwarp();
    if (lane < per) {
      const int g = mc ? (int)(cr * per + lane) : lane;  // which 4-row group of the stage
      uint32_t x = (blockIdx.x / cn) * 7919u + it * 1315423911u + g * 2654435761u;
      int r[4];
      for (int q = 0; q < 4; ++q) { x = x * 1664525u + 1013904223u; r[q] = (x >> 8) % rows; }
      uint8_t *dst = buf + s * 16384 + g * 512;
      if (mc)
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes.multicast::cluster"
            " [%0], [%1, {%2, %3, %4, %5, %6}], [%7], %8;" ::"r"(sa(dst)),
            "l"(&m1), "r"(64), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(sa(full + s)), "h"(mask)
            : "memory");
      else
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(sa(dst)),
            "l"(&m1), "r"(64), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(sa(full + s))
            : "memory");
    }
  };
  for (int it = 0; it < stages; ++it) issue(it);
  for (int it = 0; it < iters; ++it) {
    const int s = it % stages;
    wait(sa(full + s), (it / stages) & 1);
    if (lane < (int)cn) {  // free the stage in every CTA of the cluster
      uint32_t remote;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(sa(empty + s)), "r"(lane));
      asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
    }
    if (it + stages < iters) issue(it + stages);
  }
  unsigned long long t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (lane == 0) out[blockIdx.x] = t1 - t0;
}

typedef CUresult (*EncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                             const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int rows = 4000, h = 512;
  uint8_t *d;
  unsigned long long *dout;
  cudaMalloc(&d, (size_t)rows * h * 2);
  cudaMemset(d, 1, (size_t)rows * h * 2);
  cudaMalloc(&dout, 1024 * 8);
  EncodeFn enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q);
  CUtensorMap m1;
  cuuint64_t dims[2] = {(cuuint64_t)h, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)h * 2};
  cuuint32_t box1[2] = {64, 1}, es[2] = {1, 1};
  enc(&m1, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, strides, box1, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int stages = 4, iters = 512;
  const int smem = 1024 + stages * 16384 + 256;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {1, 2, 4, 8})
    for (int mc : {0, 1}) {
      if (cs == 1 && mc) continue;
      int grid = (148 / cs) * cs;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(grid);
      cfg.blockDim = dim3(32);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.attrs = at; cfg.numAttrs = 1;
      int maxc = 0;
      cudaOccupancyMaxActiveClusters(&maxc, probe, &cfg);
      grid = std::min(grid, maxc * cs);
      cfg.gridDim = dim3(grid);
      for (int rep = 0; rep < 2; ++rep) {
        cudaError_t e = cudaLaunchKernelEx(&cfg, probe, m1, rows, stages, iters, mc, dout);
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("cs %d mc %d: %s\n", cs, mc, cudaGetErrorString(e)); return 1; }
      }
      std::vector<unsigned long long> t(grid);
      cudaMemcpy(t.data(), dout, grid * 8, cudaMemcpyDeviceToHost);
      double avg = 0;
      for (auto x : t) avg += x;
      avg /= grid;
      printf("cluster %d multicast %d (grid %d, max clusters %d): per-stage %6.0f ns -> %5.1f GB/s delivered per SM\n",
             cs, mc, grid, maxc, avg / iters, 16384.0 * iters / avg);
    }
  return 0;
}
