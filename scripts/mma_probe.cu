// Probe: tcgen05.mma (kind::f16, M=128, K=16 per instruction) cadence for a small tile: NMMA MMAs
// from shared memory into NACC independent TMEM accumulators (round-robin), N = 32..256.  Reports
// ns per MMA from the first issue to the commit's mbarrier completing.  One CTA, one issuing thread.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/mma_probe.bin scripts/mma_probe.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t gtime() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint64_t desc(uint32_t saddr) {
  return (uint64_t)((saddr & 0x3FFFF) >> 4) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) |
         (2ull << 61);
}
__device__ int g_m = 128;  // MMA M (128 or 64)
__device__ __forceinline__ uint32_t idesc(int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(g_m >> 4) << 24);
}

__global__ void probe(int n, int nmma, int nacc, unsigned long long *out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t *s = (uint8_t *)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) ((uint32_t *)s)[i] = 0x3c003c00u;  // bf16 1.0
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(sa(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tslot;
  if (threadIdx.x < 32 && nacc < 0) {  // whole warp walks the loop; elect.sync picks the issuing lane
    const uint32_t id = idesc(n);
    const uint32_t abase = sa(s), bbase = sa(s + 32768);
    for (int rep = 0; rep < 2; ++rep) {
      const uint64_t t0 = gtime();
      for (int c = 0; c < nmma / 4; ++c) {
        const uint64_t ad = desc(abase + (c & 1) * 16384), bd = desc(bbase);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          asm volatile("{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm),
                       "l"(ad + 2 * k), "l"(bd + 2 * k), "r"(id), "r"((c > 0 || k > 0) ? 1u : 0u)
                       : "memory");
      }
      const uint64_t t1 = gtime();
      asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                   "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(sa(&bar))
                   : "memory");
      uint32_t ok = 0;
      while (!ok)
        asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                     : "=r"(ok) : "r"(sa(&bar)), "r"(rep & 1) : "memory");
      const uint64_t t2 = gtime();
      if (threadIdx.x == 0) { out[rep * 2] = t1 - t0; out[rep * 2 + 1] = t2 - t0; }
    }
  }
  if (threadIdx.x == 0 && nacc >= 0) {
    const uint32_t id = idesc(n);
    const uint32_t abase = sa(s), bbase = sa(s + 32768);
    const int stride = nacc ? 512 / nacc : 0;
    for (int rep = 0; rep < 2; ++rep) {
      const uint64_t t0 = gtime();
      if (nacc == 0) {  // kernel-like: 4 unrolled K steps per chunk, one accumulator
        for (int c = 0; c < nmma / 4; ++c) {
          const uint64_t ad = desc(abase + (c & 1) * 16384), bd = desc(bbase);
#pragma unroll
          for (int k = 0; k < 4; ++k)
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm),
                         "l"(ad + 2 * k), "l"(bd + 2 * k), "r"(id), "r"((c > 0 || k > 0) ? 1u : 0u)
                         : "memory");
        }
      } else {
      for (int i = 0; i < nmma; ++i) {
        const int a = i % nacc, k = (i / nacc) % 4;
        const uint64_t ad = desc(abase + ((i / 4) % 2) * 16384) + 2 * k, bd = desc(bbase) + 2 * k;
        const uint32_t acc = (i / nacc) > 0 ? 1u : 0u;
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm + a * stride),
                     "l"(ad), "l"(bd), "r"(id), "r"(acc)
                     : "memory");
      }
      }
      const uint64_t t1 = gtime();
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&bar))
                   : "memory");
      uint32_t ok = 0;
      while (!ok)
        asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                     : "=r"(ok) : "r"(sa(&bar)), "r"(rep & 1) : "memory");
      const uint64_t t2 = gtime();
      out[rep * 2] = t1 - t0;
      out[rep * 2 + 1] = t2 - t0;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

int main() {
  unsigned long long *out, h[4];
  cudaMalloc(&out, 64);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  for (int mm : {128, 64}) {
  cudaMemcpyToSymbol(g_m, &mm, sizeof(int));
  printf("M = %d\n", mm);
  for (int n : {32, 64, 80, 128, 160, 256})
    for (int nacc : {-1})
      for (int nmma : {16, 64}) {
        if (n * nacc > 512) continue;
        probe<<<1, 128, 70000>>>(n, nmma, nacc, out);
        cudaError_t e = cudaMemcpy(h, out, 32, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
        printf("N %3d acc %d mma %2d: issue %5.1f ns/mma, done %6.1f ns/mma (%.0f ns total)\n", n, nacc, nmma,
               double(h[2]) / nmma, double(h[3]) / nmma, double(h[3]));
      }
  }
  return 0;
}
