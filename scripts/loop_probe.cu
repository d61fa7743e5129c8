// Probe: per-K-chunk cadence of the operand-loader loop of ed_persistent_bf16 in isolation.
// One CTA per SM, 384 threads: warps 0-3 "epilogue" (spin on an mbarrier or park on bar.sync),
// warp 4 consumer (waits full, arrives empty), warp 5 B loader (bulk copy of bbytes per chunk),
// warps 6-11 A loaders (8-row TMA boxes or 16 B cp.async gathers, lagged release like the kernel).
// Reports ns per chunk (clock64 / SM clock) for each variant.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/loop_probe scripts/loop_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

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
__device__ __forceinline__ void arrive_tx(uint64_t *b, uint32_t n) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(n) : "memory");
}
template <int N> __device__ __forceinline__ void cpw() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

struct Cfg { int amode, rows, bbytes, D, lag, spin, fence, chunks, nwarps; };

__global__ void __launch_bounds__(384, 1) probe(const __grid_constant__ CUtensorMap m8, const __grid_constant__ CUtensorMap m128, const uint8_t *H, int nrows_tot,
                                                 const uint8_t *W, Cfg c, unsigned long long *out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t *buf = (uint8_t *)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  const uint32_t abytes = c.rows * 128, sbytes = abytes + c.bbytes;
  uint64_t *full = (uint64_t *)(buf + 196608), *empty = full + 16, *done = empty + 16;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < 16; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(full + s)), "r"(2 + c.nwarps));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(empty + s)), "r"(1));
    }
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(done)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int D = c.D;
  long long t0 = clock64();
  if (warp < 4) {
    if (c.spin) mwait(done, 0);
  } else if (warp == 4) {
    if (lane == 0) {
      for (int k = 0; k < c.chunks; ++k) {
        const int s = k % D;
        mwait(full + s, (k / D) & 1);
        arrive(empty + s);
      }
      out[blockIdx.x] = clock64() - t0;
      arrive(done);
    }
  } else if (warp == 5) {
    if (lane == 0)
      for (int k = 0; k < c.chunks; ++k) {
        const int s = k % D;
        mwait(empty + s, ((k / D) & 1) ^ 1);
        if (c.bbytes == 0) { arrive(full + s); continue; }
        arrive_tx(full + s, c.bbytes);
        const uint8_t *src = W + ((size_t)(blockIdx.x * 97 + k) * c.bbytes) % (64u << 20);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         sa(buf + s * sbytes + abytes)), "l"(src), "r"(c.bbytes), "r"(sa(full + s)) : "memory");
      }
  } else if (warp < 6 + c.nwarps) {
    const int lt = tid - 192;
    int pending = 0;
    const int base_row = (blockIdx.x * 7919) % (nrows_tot - 256);
    for (int k = 0; k < c.chunks; ++k) {
      const int s = k % D;
      mwait(empty + s, ((k / D) & 1) ^ 1);
      uint8_t *a = buf + s * sbytes;
      const int col = (k % 8) * 64;
      if (c.amode == 3) {  // one 128-row TMA box
        if (lt == 0) {
          arrive_tx(full + s, 16384);
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                  sa(a)), "l"(&m128), "r"(col), "r"(base_row + (k % 64) * 128), "r"(sa(full + s)) : "memory");
        }
      } else if (c.amode == 4) {  // 8-row TMA boxes issued one after another by lane 0
        if (lt == 0) {
          const int nbox = c.rows / 8;
          arrive_tx(full + s, abytes);
          for (int b = 0; b < nbox; ++b)
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                    sa(a + b * 1024)), "l"(&m8), "r"(col), "r"(base_row + b * 8), "r"(sa(full + s)) : "memory");
        }
      } else if (c.amode == 0) {  // 8-row TMA boxes from warp 6
        if (lt < 32) {
          const int nbox = c.rows / 8;
          if (lt == 0) arrive_tx(full + s, abytes);
          __syncwarp();
          if (lt < nbox)
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                    sa(a + lt * 1024)), "l"(&m8), "r"(col), "r"(base_row + lt * 8), "r"(sa(full + s)) : "memory");
        }
      } else if (c.amode == 2) {  // no A data
        if (lt == 0) arrive(full + s);
      } else {  // 16 B cp.async gathers of random rows
        if (lt == 0) arrive(full + s);
        for (int q = lt; q < c.rows * 8; q += 192) {
          const int r = q >> 3, ch = q & 7;
          const int gr = (base_row + r * 37 + k * 11) % nrows_tot;
          const uint8_t *src = H + ((size_t)gr * 512 + col) * 2 + ch * 16;
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa(a + r * 128 + ((ch ^ (r & 7)) << 4))), "l"(src) : "memory");
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      if (c.lag == 0) {
        __syncwarp();
        if (lane == 0) arrive(full + s);
      } else if (++pending == c.lag) {
        if (c.lag == 3) cpw<2>(); else cpw<7>();
        if (c.fence) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) arrive(full + (k + 1 - c.lag) % D);
        --pending;
      }
    }
    cpw<0>();
    __syncwarp();
    for (; pending > 0; --pending)
      if (lane == 0) arrive(full + (c.chunks - pending) % D);
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                             const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int rows = 40000, h = 512;
  uint8_t *d, *w;
  unsigned long long *dout;
  cudaMalloc(&d, (size_t)rows * h * 2);
  cudaMalloc(&w, 64u << 20);
  cudaMemset(d, 1, (size_t)rows * h * 2);
  cudaMemset(w, 2, 64u << 20);
  cudaMalloc(&dout, 1024 * 8);
  EncodeFn enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q);
  CUtensorMap m8, m128;
  cuuint64_t dims[2] = {(cuuint64_t)h, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)h * 2};
  cuuint32_t box8[2] = {64, 8}, es[2] = {1, 1};
  enc(&m8, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, strides, box8, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cuuint32_t box128[2] = {64, 128};
  enc(&m128, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, strides, box128, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int smem = 1024 + 196608 + 512;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const char *an[5] = {"tma8", "cpasync", "none", "tma128", "tma8seq"};
  std::vector<Cfg> cfgs = {
      {2, 8, 0, 14, 0, 1, 1, 256, 1}, {4, 8, 0, 14, 0, 1, 1, 256, 1}, {4, 40, 0, 3, 0, 1, 1, 256, 1},
      {4, 128, 0, 3, 0, 1, 1, 256, 1}, {0, 40, 0, 3, 0, 1, 1, 256, 1}, {3, 128, 0, 3, 0, 1, 1, 256, 1},
      {4, 8, 10240, 14, 0, 1, 1, 256, 1},
  };
  for (int grid : {1})
    for (auto c : cfgs) {
      for (int rep = 0; rep < 2; ++rep) {
        probe<<<grid, 384, smem>>>(m8, m128, d, rows, w, c, dout);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      }
      std::vector<unsigned long long> t(grid);
      cudaMemcpy(t.data(), dout, grid * 8, cudaMemcpyDeviceToHost);
      double avg = 0;
      for (auto x : t) avg += x;
      avg /= grid;
      const double ns = avg / (clk * 1e-6) / c.chunks;
      printf("grid %3d nw %d A=%-7s rows %3d B %5d D %2d lag %d spin %d fence %d : %7.1f ns/chunk  %6.1f GB/s/SM\n", grid, c.nwarps,
             an[c.amode], c.rows, c.bbytes, c.D, c.lag, c.spin, c.fence, ns, (c.rows * 128.0 + c.bbytes) / ns);
    }
  return 0;
}
