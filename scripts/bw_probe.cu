// Probe: L2 -> shared memory delivery rates on B200 for the operand shapes of the step kernel.
// Each CTA runs a ring of `stages` buffers; every stage = optional A part (gather4 of 128 random
// rows x 128 B, or one 128-row box) + optional B part (one bulk copy of bbytes).  A stage is
// re-issued as soon as its previous fill completed.  Reports per-SM and aggregate GB/s.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/bw_probe scripts/bw_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t *b, uint32_t par) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                 : "=r"(ok) : "r"(sa(b)), "r"(par) : "memory");
}

__global__ void probe(const __grid_constant__ CUtensorMap m1, const __grid_constant__ CUtensorMap m128,
                      const uint8_t *wbuf, long wbytes, const uint8_t *d_rows, int h, int rows, int amode, int bbytes, int stages, int iters,
                      unsigned long long *out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t *buf = (uint8_t *)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  const int sbytes = 16384 + 32768;
  uint64_t *bar = (uint64_t *)(buf + stages * sbytes);
  const int lane = threadIdx.x;
  if (lane == 0) {
    for (int s = 0; s < stages; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(bar + s)), "r"(amode == 3 ? blockDim.x + 1 : 1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  uint32_t seed = blockIdx.x * 7919 + 17;
  for (int it = 0; it < iters + stages; ++it) {
    const int s = it % stages;
    if (it >= stages) wait(bar + s, ((it / stages) - 1) & 1);
    __syncthreads();
    if (it >= iters) continue;
    uint8_t *a = buf + s * sbytes;
    uint8_t *b = a + 16384;
    const int abytes = (amode == 0 || amode == 3) ? 0 : 16384;
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(bar + s)), "r"(abytes + bbytes)
                   : "memory");
    __syncthreads();
    const int col = ((it * 64) % 512);
    if (amode == 3) {  // cp.async 16 B: 128 random rows x 8 chunks spread over all threads
      const int nthr = blockDim.x;
      for (int c = threadIdx.x; c < 1024; c += nthr) {
        const int r = c >> 3, ch = c & 7;
        uint32_t x = seed + it * 1315423911u + r * 2654435761u;
        x = x * 1664525u + 1013904223u;
        const int gr = (x >> 8) % rows;
        const uint8_t *src = d_rows + ((size_t)gr * h + col) * 2 + ch * 16;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa(a + r * 128 + ((ch ^ (r & 7)) << 4))), "l"(src)
                     : "memory");
      }
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(sa(bar + s)) : "memory");
    } else if (amode == 4 && lane == 0) {  // 128 single-row boxes
      uint32_t x = seed + it * 1315423911u;
      for (int r = 0; r < 128; ++r) {
        x = x * 1664525u + 1013904223u;
        const int gr = (x >> 8) % rows;
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                sa(a + r * 128)),
            "l"(&m1), "r"(col), "r"(gr), "r"(sa(bar + s))
            : "memory");
      }
    } else if (amode == 1) {  // 32 gather4 of random rows
      uint32_t x = seed + it * 1315423911u + lane * 2654435761u;
      int r[4];
      for (int q = 0; q < 4; ++q) { x = x * 1664525u + 1013904223u; r[q] = (x >> 8) % rows; }
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
          "%4, %5, %6}], [%7];" ::"r"(sa(a + lane * 512)),
          "l"(&m1), "r"(col), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(sa(bar + s))
          : "memory");
    } else if (amode == 2 && lane == 0) {  // one 128-row box
      int r0 = ((seed + it * 977) % (rows - 128));
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
              sa(a)),
          "l"(&m128), "r"(col), "r"(r0), "r"(sa(bar + s))
          : "memory");
    }
    if (bbytes > 0 && lane == 0) {
      long off = ((long)(blockIdx.x % 16) * 20 * 32768L + (long)(it % 64) * 81920L) % (wbytes - bbytes);
      off &= ~127L;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       sa(b)),
                   "l"(wbuf + off), "r"(bbytes), "r"(sa(bar + s))
                   : "memory");
    }
  }
  unsigned long long t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (lane == 0) out[blockIdx.x] = t1 - t0;
}

typedef CUresult (*EncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                             const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int rows = 4000, h = 512;
  const long wbytes = 5L << 20;
  uint8_t *d, *w;
  unsigned long long *dout;
  cudaMalloc(&d, (size_t)rows * h * 2);
  cudaMalloc(&w, wbytes);
  cudaMemset(d, 1, (size_t)rows * h * 2);
  cudaMemset(w, 2, wbytes);
  cudaMalloc(&dout, 1024 * 8);
  EncodeFn enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q);
  CUtensorMap m1, m128;
  cuuint64_t dims[2] = {(cuuint64_t)h, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)h * 2};
  cuuint32_t box1[2] = {64, 1}, box128[2] = {64, 128}, es[2] = {1, 1};
  enc(&m1, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, strides, box1, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  enc(&m128, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, strides, box128, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int smem = 1024 + 4 * (16384 + 32768) + 64;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char *an[5] = {"none", "gather4", "box128", "cpasync", "rowbox"};
  struct Cfg { int amode, bbytes, stages, grid, threads; };
  std::vector<Cfg> cfgs;
  for (int grid : {148})
    for (int st : {4})
      for (int am : {3, 4})
        for (int bb : {0, 20480})
          for (int th : {32, 64, 128, 256})
            if (am == 3 || th == 32) cfgs.push_back({am, bb, st, grid, th});
  for (auto c : cfgs) {
    const int iters = 256;
    for (int rep = 0; rep < 2; ++rep) {
      probe<<<c.grid, c.threads, smem>>>(m1, m128, w, wbytes, d, h, rows, c.amode, c.bbytes, c.stages, iters, dout);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    }
    std::vector<unsigned long long> t(c.grid);
    cudaMemcpy(t.data(), dout, c.grid * 8, cudaMemcpyDeviceToHost);
    double mx = 0, avg = 0;
    for (auto x : t) { mx = x > mx ? x : mx; avg += x; }
    avg /= c.grid;
    const double bytes = (double)iters * ((c.amode ? 16384 : 0) + c.bbytes);
    printf("threads %3d ", c.threads);
    printf("grid %3d stages %d A=%-7s B=%5d : per-stage %7.0f ns, per-SM %6.1f GB/s, aggregate %7.0f GB/s\n", c.grid,
           c.stages, an[c.amode], c.bbytes, avg / iters, bytes / avg, bytes * c.grid / mx);
  }
  return 0;
}
