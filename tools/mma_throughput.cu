// Microbenchmark: tcgen05.mma cost vs N and vs the number of independent
// accumulation chains in flight (1 CTA, one issuing thread).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_throughput tools/mma_throughput.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2605_18052_b200/csrc/tc_ptx.cuh"
using namespace dmv3d;

__global__ void k(int iters, int ksteps, int n, int chains, long long *out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t *A = sm, *B = sm + 128 * 128 * 2;  // A: 128 x 128 fp16, B: 256 x 128 fp16
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  for (int i = threadIdx.x; i < 128 * 128 * 2 + 256 * 128 * 2; i += blockDim.x) sm[i] = 0;
  if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
  if (threadIdx.x < 32) ptx::tmem_alloc(&tbase, 512);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t idesc = ptx::idesc_f16(128, n, 0);
  uint32_t phase = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (threadIdx.x == 0) {
      ptx::tc_fence_after();
      for (int ks = 0; ks < ksteps; ++ks)
        for (int c = 0; c < chains; ++c) {
          const uint64_t ad = ptx::smem_desc(ptx::smem_u32(A) + ks * 256, 128, 2048, 0);
          const uint64_t bd = ptx::smem_desc(ptx::smem_u32(B) + ks * 256, 128, 2048, 0);
          ptx::mma_f16_ss(tbase + c * n, ad, bd, idesc, ks > 0);
        }
      ptx::mma_commit(&bar);
    }
    ptx::mbar_wait(&bar, phase);
    phase ^= 1u;
    ptx::tc_fence_after();
    ptx::tc_fence_before();
    ptx::bar_sync(1, blockDim.x);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
  ptx::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) { ptx::tc_fence_after(); ptx::tmem_dealloc(tbase, 512); }
}

int main() {
  long long *d, h;
  cudaMalloc(&d, 8);
  const int smem = 128 * 128 * 2 + 256 * 128 * 2 + 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int n : {64, 128, 256})
    for (int chains : {1, 2, 4})
      for (int ks : {1, 8}) {
        if (chains * n > 512) continue;
        k<<<1, 128, smem>>>(1000, ks, n, chains, d);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("N=%3d chains=%d ksteps=%d : %5lld cycles/round trip  (%s)\n", n, chains, ks, h,
               cudaGetErrorString(e));
      }
  return 0;
}
