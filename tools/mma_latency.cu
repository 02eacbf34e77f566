// Microbenchmark: round-trip latency of a tcgen05.mma chain (issue -> commit ->
// mbarrier wait) on one SM, as used per layer by render_tc_kernel.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_latency tools/mma_latency.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2605_18052_b200/csrc/tc_ptx.cuh"

using namespace dmv3d;

__global__ void k(int iters, int ksteps, int n, int a_tmem, long long *out) {
  __shared__ __align__(1024) uint8_t A[128 * 80 * 2];
  __shared__ __align__(1024) uint8_t B[64 * 128 * 2];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  for (int i = threadIdx.x; i < (int)sizeof(A); i += blockDim.x) A[i] = 0;
  for (int i = threadIdx.x; i < (int)sizeof(B); i += blockDim.x) B[i] = 0;
  if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
  if (threadIdx.x < 32) ptx::tmem_alloc(&tbase, 256);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tbase;
  const uint32_t idesc = ptx::idesc_f16(128, n, 0);
  uint32_t phase = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (threadIdx.x == 0) {
      ptx::tc_fence_after();
      for (int ks = 0; ks < ksteps; ++ks) {
        const uint64_t bd = ptx::smem_desc(ptx::smem_u32(B) + ks * 256, 128, 1280, 0);
        if (a_tmem) {
          ptx::mma_f16_ts(tmem, tmem + 128 + ks * 8, bd, idesc, ks > 0);
        } else {
          const uint64_t ad = ptx::smem_desc(ptx::smem_u32(A) + ks * 256, 128, 1280, 0);
          ptx::mma_f16_ss(tmem, ad, bd, idesc, ks > 0);
        }
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
  if (threadIdx.x < 32) { ptx::tc_fence_after(); ptx::tmem_dealloc(tbase, 256); }
}

int main() {
  long long *d, h;
  cudaMalloc(&d, 8);
  for (int a_tmem = 0; a_tmem < 2; ++a_tmem)
    for (int ks : {1, 4, 5, 8})
      for (int n : {16, 64}) {
        k<<<1, 128>>>(2000, ks, n, a_tmem, d);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("A_%s ksteps=%d N=%d : %lld cycles per round trip (%s)\n", a_tmem ? "tmem" : "smem",
               ks, n, h, cudaGetErrorString(e));
      }
  return 0;
}
