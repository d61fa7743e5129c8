// Probe: does cp.async.mbarrier.arrive.noinc serialise a thread's later cp.async behind the earlier
// ones?  One CTA, one loader warp (8 active lanes: one 128 B row per chunk, like a one-row tile) and a
// consumer thread; NCH chunks through a 4-stage ring.  Variants:
//   0: per chunk 8 x cp.async 16 B + cp.async.mbarrier.arrive.noinc on the chunk's full barrier
//   1: same loads, no per-chunk arrive: one commit + wait_group 0 at the end (pure issue time)
//   2: per chunk cp.async + commit_group; full barrier arrived after wait_group 0 (serialised)
// Reports ns from first issue to the consumer seeing the last chunk, and the issue time of the loop.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/arrive_probe scripts/arrive_probe.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mwait(uint64_t *b, uint32_t par) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                 : "=r"(ok) : "r"(sa(b)), "r"(par) : "memory");
}
__device__ __forceinline__ void arrive(uint64_t *b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory");
}
__device__ __forceinline__ void cp16(uint32_t d, const void *s) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(s) : "memory");
}
__device__ __forceinline__ uint64_t gtime() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

constexpr int kStages = 4;

__global__ void probe(const uint8_t *src, int nch, int variant, int stride, unsigned long long *out) {
  __shared__ __align__(1024) uint8_t st[kStages][8192];
  __shared__ uint64_t full[kStages], empty[kStages];
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(full + s)), "r"(variant >= 3 ? 33 : 32));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(empty + s)), "r"(1));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid < 32) {
    const uint64_t t0 = gtime();
    for (int c = 0; c < nch; ++c) {
      const int s = c % kStages;
      mwait(empty + s, ((c / kStages) & 1) ^ 1);
      if (variant == 3 && tid == 0) arrive(full + s);
      if (variant == 4 && tid == 0)
        asm volatile("mbarrier.arrive.relaxed.cta.shared::cta.b64 _, [%0];" ::"r"(sa(full + s)) : "memory");
      if (tid < 8) cp16(sa(&st[s][tid * 16]), src + (size_t)c * stride + tid * 16);
      if (variant == 0 || variant >= 3) {
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(sa(full + s)) : "memory");
      } else if (variant == 1) {
        arrive(full + s);  // data not awaited (issue-rate probe only)
      } else {
        asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
        arrive(full + s);
      }
    }
    const uint64_t t1 = gtime();
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
    if (tid == 0) { out[0] = t0; out[1] = t1; }
  } else if (tid == 32) {
    for (int c = 0; c < nch; ++c) {
      const int s = c % kStages;
      mwait(full + s, (c / kStages) & 1);
      arrive(empty + s);
    }
    out[2] = gtime();
  }
}

// Issue-rate probe: lane l < act issues n cp.async 16 B (distinct lines, cold in L2 when cold != 0),
// timestamps before / after the issue loop and after wait_group 0.
__global__ void issue_probe(const uint8_t *src, int n, int act, unsigned long long *out) {
  __shared__ __align__(1024) uint8_t buf[32768];
  const int tid = threadIdx.x;
  if (tid < act) {
    const uint64_t t0 = gtime();
    for (int i = 0; i < n; ++i)
      cp16(sa(&buf[((i * act + tid) * 16) & 32767]), src + ((size_t)i * act + tid) * 4096);
    const uint64_t t1 = gtime();
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
    const uint64_t t2 = gtime();
    if (tid == 0) { out[0] = t0; out[1] = t1; out[2] = t2; }
  }
}
__global__ void flush(uint8_t *p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n / 16; i += (size_t)gridDim.x * blockDim.x)
    reinterpret_cast<uint4 *>(p)[i] = make_uint4(i, 0, 0, 0);
}

int main() {
  const int nch = 64, stride = 1 << 16;
  uint8_t *src;
  unsigned long long *out, h[3];
  cudaMalloc(&src, (size_t)nch * stride + 4096);
  cudaMemset(src, 1, (size_t)nch * stride + 4096);
  cudaMalloc(&out, 64);
  for (int variant = 0; variant < 5; ++variant)
    for (int rep = 0; rep < 3; ++rep) {
      cudaMemset(src + (rep == 2 ? 0 : 0), rep, 64);  // rows just written by the host copy engine
      probe<<<1, 64>>>(src, nch, variant, stride, out);
      cudaMemcpy(h, out, 24, cudaMemcpyDeviceToHost);
      printf("variant %d: issue %.0f ns/chunk, done %.0f ns/chunk\n", variant, double(h[1] - h[0]) / nch,
             double(h[2] - h[0]) / nch);
    }
  uint8_t *big, *fl;
  cudaMalloc(&big, (size_t)1 << 30);
  cudaMemset(big, 1, (size_t)1 << 30);
  cudaMalloc(&fl, (size_t)512 << 20);
  for (int act : {1, 8, 32})
    for (int n : {1, 2, 4, 8, 16, 32, 64})
      for (int cold = 0; cold < 2; ++cold) {
        if (cold) flush<<<592, 512>>>(fl, (size_t)512 << 20);
        else issue_probe<<<1, 32>>>(big, n, act, out);
        issue_probe<<<1, 32>>>(big, n, act, out);
        cudaMemcpy(h, out, 24, cudaMemcpyDeviceToHost);
        printf("act %2d n %2d %s: issue %6.0f ns, complete %6.0f ns\n", act, n, cold ? "cold" : "warm",
               double(h[1] - h[0]), double(h[2] - h[0]));
      }
  return 0;
}
