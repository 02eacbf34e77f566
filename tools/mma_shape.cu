// Microbenchmark: round trip of an MMA chain per instruction shape -- the render kernel's
// M = 128, N = 64 (A from TMEM or smem) against the transposed-MLP shape M = 64, N = 256
// (A = weights in smem, B = activations^T in smem), 1 or 3 issuing groups per SM, all SMs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_shape tools/mma_shape.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2605_18052_b200/csrc/tc_ptx.cuh"

using namespace dmv3d;

__global__ void k(int iters, int steps, int M, int N, int a_tmem, long long *out) {
  extern __shared__ __align__(1024) uint8_t sm[];  // A: 128 x 128 fp16 (32 KB), B: 256 x 128 (64 KB)
  uint8_t *A = sm, *B = sm + 32768;
  __shared__ uint64_t bar[4];
  __shared__ uint32_t tbase;
  const int g = threadIdx.x >> 7, tid = threadIdx.x & 127;
  for (int i = threadIdx.x; i < 32768 + 65536; i += blockDim.x) sm[i] = 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) ptx::mbar_init(&bar[i], 1);
    ptx::fence_mbar_init();
  }
  if (threadIdx.x < 32) ptx::tmem_alloc(&tbase, 512);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tbase + (uint32_t)g * 160u;  // D at +0 (<= 256 cols for g = 0 only when N = 256)
  const uint32_t idesc = ptx::idesc_f16(M, N, 0);
  uint32_t phase = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (tid == 0) {
      ptx::tc_fence_after();
      for (int ks = 0; ks < steps; ++ks) {
        // K-major no-swizzle core matrices: LBO = 128 B (K direction), SBO = 16 * ... rows
        const uint64_t bd = ptx::smem_desc(ptx::smem_u32(B) + (ks & 3) * 256, 128, 2048, 0);
        if (a_tmem) {
          ptx::mma_f16_ts(tmem, tmem + 128 + (ks & 3) * 8, bd, idesc, ks > 0);
        } else {
          const uint64_t ad = ptx::smem_desc(ptx::smem_u32(A) + (ks & 3) * 256, 128, 2048, 0);
          ptx::mma_f16_ss(tmem, ad, bd, idesc, ks > 0);
        }
      }
      ptx::mma_commit(&bar[g]);
    }
    ptx::mbar_wait(&bar[g], phase);
    phase ^= 1u;
    ptx::tc_fence_after();
    ptx::tc_fence_before();
    ptx::bar_sync(1 + g, 128);
  }
  long long t1 = clock64();
  if (tid == 0 && blockIdx.x == 0) out[g] = (t1 - t0) / iters;
  ptx::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tbase, 512);
  }
}

int main() {
  long long *d, h[4];
  cudaMalloc(&d, 32);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768 + 65536 + 1024);
  printf("groups   M    N  a_tmem steps | round-trip cycles (group 0)  per MMA\n");
  struct S { int M, N, at; } shapes[] = {{128, 64, 1}, {128, 64, 0}, {64, 256, 0}, {128, 256, 0},
                                         {64, 128, 0}, {128, 128, 0}};
  for (int groups : {1, 3})
    for (auto sh : shapes)
      for (int steps : {1, 4, 5}) {
        if (groups == 3 && sh.N == 256) continue;  // TMEM: 3 x 256 columns do not fit
        cudaMemset(d, 0, 32);
        k<<<148, 128 * groups, 32768 + 65536 + 1024>>>(2000, steps, sh.M, sh.N, sh.at, d);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
        cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
        printf("%6d %4d %4d %6d %5d | %10lld  %8.0f\n", groups, sh.M, sh.N, sh.at, steps, h[0],
               (double)h[0] / steps);
      }
  return 0;
}
