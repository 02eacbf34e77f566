// Microbenchmark: tcgen05.mma throughput with G independent issuing groups per CTA
// (one CTA per SM, like render_tc_kernel): group g (128 threads) issues a chain of
// `ks` K = 16 steps into its own TMEM region, commits to its own mbarrier and waits.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mma_groups tools/mma_groups.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2605_18052_b200/csrc/tc_ptx.cuh"
using namespace dmv3d;

__global__ void k(int iters, int ksteps, int n, int ts, int mm, long long *out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *A = sm, *B = sm + 128 * 128 * 2;
  __shared__ uint64_t bar[8];
  __shared__ uint32_t tbase;
  const int G = blockDim.x / 128, g = threadIdx.x / 128, tid = threadIdx.x % 128;
  for (int i = threadIdx.x; i < 128 * 128 * 2 + 256 * 128 * 2; i += blockDim.x) sm[i] = 0;
  if (threadIdx.x == 0) { for (int i = 0; i < 8; ++i) ptx::mbar_init(&bar[i], 1); ptx::fence_mbar_init(); }
  if (threadIdx.x < 32) ptx::tmem_alloc(&tbase, 512);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t idesc = ptx::idesc_f16(mm, n, 0);
  const uint32_t d = tbase + (uint32_t)(g * (512 / G));  // group region (D then A for TS)
  uint32_t phase = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (tid == 0) {
      ptx::tc_fence_after();
      for (int ks = 0; ks < ksteps; ++ks) {
        const uint64_t ad = ptx::smem_desc(ptx::smem_u32(A) + ks * 256, 128, 2048, 0);
        const uint64_t bd = ptx::smem_desc(ptx::smem_u32(B) + ks * 256, 128, 2048, 0);
        if (ts)  // A from TMEM: 8 columns per K = 16 step, just after this group's D
          ptx::mma_f16_ts(d, d + (uint32_t)n + ks * 8, bd, idesc, ks > 0);
        else
          ptx::mma_f16_ss(d, ad, bd, idesc, ks > 0);
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
  if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
  ptx::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) { ptx::tc_fence_after(); ptx::tmem_dealloc(tbase, 512); }
}

int main() {
  long long *d, h;
  cudaMalloc(&d, 8);
  const int smem = 128 * 128 * 2 + 256 * 128 * 2 + 2048;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int mm : {128, 64})
    for (int n : {64, 128, 256})
      for (int G : {1, 2, 4})
        for (int ks : {1, 8}) {
          const int ts = 0;
          if (G * n > 512) continue;
          k<<<148, 128 * G, smem>>>(2000, ks, n, ts, mm, d);
          cudaError_t e = cudaDeviceSynchronize();
          cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
          printf("SS M=%3d N=%3d groups=%d ksteps=%d : %5lld cycles/round  %.1f cycles/MMA per SM  (%s)\n",
                 mm, n, G, ks, h, (double)h / (G * ks), cudaGetErrorString(e));
          if (e != cudaSuccess) return 1;
        }
  return 0;
}
