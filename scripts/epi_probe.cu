// Probe: cost of one 8-unit TreeLSTM-internal epilogue pass (the persistent kernel's umma_epilogue)
// for 4 warps (one per SM sub-partition), split into its parts: TMEM loads, gate math (MUFU tanh),
// global stores.  Variants: 0 = full pass; 1 = no stores; 2 = no MUFU (FMA stand-ins); 3 = stores
// only; 4 = full pass with tanh.approx.f16x2 (two gates per MUFU op).  Reports cycles per pass
// (clock64, warp 0 lane 0, median over passes).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/epi_probe.bin scripts/epi_probe.cu
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ float tanh_fast(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float sig_fast(float x) { return fmaf(0.5f, tanh_fast(0.5f * x), 0.5f); }
__device__ __forceinline__ uint32_t tanh_h2(uint32_t x) {
  uint32_t y;
  asm("tanh.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float *v) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
  for (int k = 0; k < 8; ++k) v[k] = __uint_as_float(r[k]);
}

__global__ void __launch_bounds__(128, 1) probe(int variant, int npass, __nv_bfloat16 *H, float *C, const float *Cin,
                                                long long *out, int one_warp) {
  __shared__ uint32_t tslot;
  __shared__ float sbias[5 * 512];
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int q = tid; q < 5 * 512; q += 128) sbias[q] = 0.01f * (q % 7);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(sa(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tacc = tslot + ((uint32_t)(warp * 32) << 16);
  const int h = 512;
  const int row = blockIdx.x * 128 + tid;
  long long t_sum[16];
  float keep = 0.f;
  const float4 *clp = reinterpret_cast<const float4 *>(Cin + (size_t)row * h);
  const float4 c0 = clp[0], c1 = clp[1];  // child c: loaded before the timed passes (as prefetched)
  keep += c0.x;
  for (int sp = 0; sp < (one_warp && warp > 0 ? 0 : npass); ++sp) {
    const long long t0 = clock64();
    const int j0 = (sp % 6) * 8;
    float z[5][8];
    if (variant != 3 && variant != 5) {
      for (int g = 0; g < 5; ++g) tmem_ld8(tacc + (uint32_t)(g * 16 + (sp & 1) * 8), z[g]);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    } else {
      for (int g = 0; g < 5; ++g)
        for (int k = 0; k < 8; ++k) z[g][k] = 0.1f * (g + k + sp);
    }
    const float aux0[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
    float hv[8], cv[8];
    for (int g = 0; g < 5; ++g)
      for (int k = 0; k < 8; ++k) z[g][k] += sbias[g * h + j0 + k];
    if (variant == 6) {
      for (int k = 0; k < 8; ++k) { cv[k] = z[0][k]; hv[k] = z[1][k]; }
    } else if (variant == 2 || variant == 5) {
      for (int k = 0; k < 8; ++k) {
        cv[k] = fmaf(z[0][k], z[4][k], fmaf(z[1][k], aux0[k], z[2][k] * aux0[k]));
        hv[k] = z[3][k] * cv[k];
      }
    } else if (variant == 4) {
      for (int k = 0; k < 8; k += 2) {
        // sigmoids of i, fl, fr, o (pairs of units) and tanh(u) as f16x2
        float a[2][5];
        for (int g = 0; g < 5; ++g) {
          __half2 x = __floats2half2_rn(g == 4 ? z[g][k] : 0.5f * z[g][k], g == 4 ? z[g][k + 1] : 0.5f * z[g][k + 1]);
          uint32_t y = tanh_h2(*reinterpret_cast<uint32_t *>(&x));
          float2 f = __half22float2(*reinterpret_cast<__half2 *>(&y));
          a[0][g] = g == 4 ? f.x : fmaf(0.5f, f.x, 0.5f);
          a[1][g] = g == 4 ? f.y : fmaf(0.5f, f.y, 0.5f);
        }
        for (int u = 0; u < 2; ++u) cv[k + u] = a[u][0] * a[u][4] + a[u][1] * aux0[k + u] + a[u][2] * aux0[k + u];
        __half2 cx = __floats2half2_rn(cv[k], cv[k + 1]);
        uint32_t ty = tanh_h2(*reinterpret_cast<uint32_t *>(&cx));
        float2 tf = __half22float2(*reinterpret_cast<__half2 *>(&ty));
        hv[k] = a[0][3] * tf.x;
        hv[k + 1] = a[1][3] * tf.y;
      }
    } else {
      for (int k = 0; k < 8; ++k) {
        cv[k] = sig_fast(z[0][k]) * tanh_fast(z[4][k]) + sig_fast(z[1][k]) * aux0[k] + sig_fast(z[2][k]) * aux0[k];
        hv[k] = sig_fast(z[3][k]) * tanh_fast(cv[k]);
      }
    }
    if (variant != 1 && variant != 5 && variant != 6) {
      uint32_t packed[4];
      for (int k = 0; k < 4; ++k) {
        __nv_bfloat162 t = __floats2bfloat162_rn(hv[2 * k], hv[2 * k + 1]);
        packed[k] = *reinterpret_cast<uint32_t *>(&t);
      }
      *reinterpret_cast<uint4 *>(H + (size_t)row * h + j0) = make_uint4(packed[0], packed[1], packed[2], packed[3]);
      float4 *cd = reinterpret_cast<float4 *>(C + (size_t)row * h + j0);
      cd[0] = make_float4(cv[0], cv[1], cv[2], cv[3]);
      cd[1] = make_float4(cv[4], cv[5], cv[6], cv[7]);
    } else {
      for (int k = 0; k < 8; ++k) keep += hv[k] + cv[k];
    }
    const long long t1 = clock64();
    if (sp < 16) t_sum[sp] = t1 - t0;
  }
  if (tid == 0)
    for (int sp = 0; sp < 16 && sp < npass; ++sp) out[blockIdx.x * 16 + sp] = t_sum[sp];
  if (keep == 12345.f) out[0] = 0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tslot));
}

int main() {
  const int grid = 148, h = 512;
  __nv_bfloat16 *H;
  float *C, *Cin;
  long long *out, hout[148 * 16];
  cudaMalloc(&H, (size_t)grid * 128 * h * 2);
  cudaMalloc(&C, (size_t)grid * 128 * h * 4);
  cudaMalloc(&Cin, (size_t)grid * 128 * h * 4);
  cudaMemset(Cin, 0, (size_t)grid * 128 * h * 4);
  cudaMalloc(&out, sizeof(hout));
  const char *names[] = {"full pass", "no stores", "no MUFU", "stores+math, no TMEM", "f16x2 tanh",
                         "bias+FMA only", "TMEM ld only"};
  for (int ow = 0; ow < 2; ++ow)
  for (int v = 0; v < 7; ++v) {
    for (int rep = 0; rep < 2; ++rep) probe<<<grid, 128>>>(v, 12, H, C, Cin, out, ow);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("%s: %s\n", names[v], cudaGetErrorString(e)); return 1; }
    cudaMemcpy(hout, out, sizeof(hout), cudaMemcpyDeviceToHost);
    printf("%s %-22s cycles per pass (CTA 0, passes 0..11):", ow ? "1 warp " : "4 warps", names[v]);
    for (int sp = 0; sp < 12; ++sp) printf(" %lld", hout[sp]);
    printf("\n");
  }
  return 0;
}
