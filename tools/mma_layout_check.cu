// Numerical check of the SWIZZLE_NONE MN-major shared-memory descriptor convention
// the tensor-core backward relies on (1 CTA, M = 128, N = 64, K = 32 in two K = 16
// steps, exact small-integer fp16 operands).  Core matrix = 8 rows x 16 B; for an
// MN-major operand a core matrix holds 8 K-rows of 8 contiguous M (or N) elements.
// Hypothesis H1: as for K-major, LBO = stride between core matrices along K and
// SBO = stride along M/N.  Each case prints the max error for H1 and for the swap.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/mma_layout_check tools/mma_layout_check.cu
#include <cstdint>
#include <cstdio>
#include <cmath>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include "../paper_2605_18052_b200/csrc/tc_ptx.cuh"
using namespace dmv3d;

constexpr int M = 128, N = 64, K = 32;

__host__ __device__ inline float aval(int m, int k) { return (float)(((m * 3 + k * 7) % 11) - 5); }
__host__ __device__ inline float bval(int k, int n) { return (float)(((k * 5 + n * 3) % 7) - 3); }

// a_mn / b_mn: operand stored MN-major; swap: exchange LBO and SBO of that operand
__global__ void kern(int a_mn, int b_mn, int swap, float *out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *A = sm, *B = sm + M * K * 2;
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int t = threadIdx.x;
  // A [M][K]
  for (int e = t; e < M * K; e += blockDim.x) {
    const int m = e / K, k = e % K;
    uint32_t off;
    if (a_mn) off = (k >> 3) * ((M / 8) * 128) + (m >> 3) * 128 + (k & 7) * 16 + (m & 7) * 2;
    else off = (m >> 3) * ((K / 8) * 128) + (k >> 3) * 128 + (m & 7) * 16 + (k & 7) * 2;
    *reinterpret_cast<__half *>(A + off) = __float2half(aval(m, k));
  }
  // B [K][N]
  for (int e = t; e < K * N; e += blockDim.x) {
    const int k = e / N, n = e % N;
    uint32_t off;
    if (b_mn) off = (k >> 3) * ((N / 8) * 128) + (n >> 3) * 128 + (k & 7) * 16 + (n & 7) * 2;
    else off = (n >> 3) * ((K / 8) * 128) + (k >> 3) * 128 + (n & 7) * 16 + (k & 7) * 2;
    *reinterpret_cast<__half *>(B + off) = __float2half(bval(k, n));
  }
  if (t == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
  if (t < 32) ptx::tmem_alloc(&tbase, 64);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t idesc = ptx::idesc_f16(M, N, b_mn) | ((uint32_t)a_mn << 15);
  if (t == 0) {
    for (int ks = 0; ks < K / 16; ++ks) {
      uint64_t ad, bd;
      if (a_mn) {  // K stride 2048, M stride 128; a K = 16 step = 2 K core matrices
        const uint32_t kst = (M / 8) * 128, mst = 128;
        ad = ptx::smem_desc(ptx::smem_u32(A) + ks * 2 * kst, swap ? mst : kst, swap ? kst : mst, 0);
      } else {
        ad = ptx::smem_desc(ptx::smem_u32(A) + ks * 256, 128, (K / 8) * 128, 0);
      }
      if (b_mn) {
        const uint32_t kst = (N / 8) * 128, nst = 128;
        bd = ptx::smem_desc(ptx::smem_u32(B) + ks * 2 * kst, swap ? nst : kst, swap ? kst : nst, 0);
      } else {
        bd = ptx::smem_desc(ptx::smem_u32(B) + ks * 256, 128, (K / 8) * 128, 0);
      }
      ptx::mma_f16_ss(tbase, ad, bd, idesc, ks > 0);
    }
    ptx::mma_commit(&bar);
  }
  ptx::mbar_wait(&bar, 0);
  ptx::tc_fence_after();
  uint32_t v[32];
  for (int h = 0; h < 2; ++h) {
    ptx::tmem_ld32(tbase + ((uint32_t)((t >> 5) * 32) << 16) + 32 * h, v);
    ptx::tmem_ld_wait();
    for (int c = 0; c < 32; ++c) out[t * N + 32 * h + c] = __uint_as_float(v[c]);
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (t < 32) { ptx::tc_fence_after(); ptx::tmem_dealloc(tbase, 64); }
}

int main() {
  float *d;
  cudaMalloc(&d, M * N * 4);
  float h[M * N];
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  const char *names[3] = {"A K-major, B MN-major", "A MN-major, B K-major", "A MN-major, B MN-major"};
  const int cases[3][2] = {{0, 1}, {1, 0}, {1, 1}};
  for (int c = 0; c < 3; ++c)
    for (int swap = 0; swap < 2; ++swap) {
      cudaMemset(d, 0, M * N * 4);
      kern<<<1, 128, 64 * 1024>>>(cases[c][0], cases[c][1], swap, d);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double err = 0;
      for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n) {
          double ref = 0;
          for (int k = 0; k < K; ++k) ref += aval(m, k) * bval(k, n);
          err = fmax(err, fabs(ref - h[m * N + n]));
        }
      printf("%-24s %s: max err %g (%s)\n", names[c], swap ? "swapped (LBO=MN, SBO=K)" : "H1 (LBO=K, SBO=MN)",
             err, cudaGetErrorString(e));
    }
  return 0;
}
