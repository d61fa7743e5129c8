// Probe: TMA tile::gather4 and single-row tile loads into a 128B-swizzled K-major tile (sm_100a).
// nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/tma_probe scripts/tma_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(const __grid_constant__ CUtensorMap m1, const __grid_constant__ CUtensorMap m128,
                      int mode, uint16_t *out) {
  __shared__ __align__(1024) uint16_t tile[128 * 64];
  __shared__ __align__(8) uint64_t bar;
  for (int i = threadIdx.x; i < 128 * 64; i += blockDim.x) tile[i] = 0xFFFF;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  asm volatile("fence.proxy.async.shared::cta;");
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(128 * 128));
    if (mode == 0) {  // 32 gather4: rows r of the tile <- global row (7*r + 3) % 300, column chunk 64
      for (int g = 0; g < 32; ++g) {
        int r0 = (7 * (4 * g + 0) + 3) % 300, r1 = (7 * (4 * g + 1) + 3) % 300;
        int r2 = (7 * (4 * g + 2) + 3) % 300, r3 = (7 * (4 * g + 3) + 3) % 300;
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::
                "r"(sa(tile + g * 4 * 64)), "l"(&m1), "r"(64), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(sa(&bar))
            : "memory");
      }
    } else if (mode == 1) {  // 128 single-row tile loads
      for (int r = 0; r < 128; ++r) {
        int gr = (7 * r + 3) % 300;
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                sa(tile + r * 64)),
            "l"(&m1), "r"(64), "r"(gr), "r"(sa(&bar))
            : "memory");
      }
    } else {  // one 128-row box starting at row 250 (rows >= 300 are out of bounds -> zero)
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
              sa(tile)),
          "l"(&m128), "r"(64), "r"(250), "r"(sa(&bar))
          : "memory");
    }
  }
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p;}"
                 : "=r"(ok) : "r"(sa(&bar)) : "memory");
  __syncthreads();
  for (int i = threadIdx.x; i < 128 * 64; i += blockDim.x) out[i] = tile[i];
}

typedef CUresult (*EncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                             const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int rows = 300, h = 256;
  std::vector<uint16_t> hbuf(rows * h);
  for (int r = 0; r < rows; ++r)
    for (int k = 0; k < h; ++k) hbuf[r * h + k] = (uint16_t)((r * 7 + k * 13) & 0x7fff);
  uint16_t *d, *dout;
  cudaMalloc(&d, rows * h * 2);
  cudaMalloc(&dout, 128 * 64 * 2);
  cudaMemcpy(d, hbuf.data(), rows * h * 2, cudaMemcpyHostToDevice);
  EncodeFn enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q);
  CUtensorMap m1, m128;
  cuuint64_t dims[2] = {(cuuint64_t)h, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)h * 2};
  cuuint32_t box1[2] = {64, 1}, box128[2] = {64, 128}, es[2] = {1, 1};
  CUresult r1 = enc(&m1, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, strides, box1, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUresult r2 = enc(&m128, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, strides, box128, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode box{64,1}=%d box{64,128}=%d\n", (int)r1, (int)r2);
  for (int mode = 0; mode < 3; ++mode) {
    probe<<<1, 128>>>(m1, m128, mode, dout);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("mode %d: CUDA error %s\n", mode, cudaGetErrorString(e)); return 1; }
    std::vector<uint16_t> o(128 * 64);
    cudaMemcpy(o.data(), dout, 128 * 64 * 2, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int r = 0; r < 128; ++r)
      for (int k = 0; k < 64; ++k) {
        int gr = mode < 2 ? (7 * r + 3) % 300 : 250 + r;
        uint16_t expect = gr < rows ? hbuf[gr * h + 64 + k] : 0;
        int ch = k / 8, e8 = k % 8;
        uint16_t got = o[r * 64 + ((ch ^ (r & 7)) * 8) + e8];
        if (got != expect) ++bad;
      }
    printf("mode %d (%s): %s (%d mismatches)\n", mode, mode == 0 ? "gather4" : mode == 1 ? "row tiles" : "128-row box",
           bad ? "FAIL" : "PASS", bad);
  }
  return 0;
}
