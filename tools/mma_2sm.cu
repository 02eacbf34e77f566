// Microbenchmark: pipe cost of CTA-pair tcgen05.mma (cta_group::2, M = 256) vs the
// single-SM form, with G issuing groups per CTA (74 clusters of 2 CTAs = 148 SMs).
// The leader CTA's group g issues `ks` K = 16 steps into its TMEM region, commits with a
// multicast arrive to both CTAs' mbarrier g; both CTAs wait.  Also times a cross-CTA
// handshake per round (the peer's 128 threads arrive on the leader's barrier).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mma_2sm tools/mma_2sm.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2605_18052_b200/csrc/tc_ptx.cuh"
using namespace dmv3d;

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// arrive on the mbarrier at the same smem offset in CTA `rank` of the cluster
__device__ __forceinline__ void mbar_arrive_remote(uint64_t *bar, uint32_t rank) {
  asm volatile(
      "{\n\t.reg .b32 ra;\n\t"
      "mapa.shared::cluster.u32 ra, %0, %1;\n\t"
      "mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n\t}" ::"r"(ptx::smem_u32(bar)),
      "r"(rank)
      : "memory");
}

__global__ void __cluster_dims__(2, 1, 1)
    k2(int iters, int ksteps, int n, int handshake, long long *out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *A = sm, *B = sm + 128 * 128 * 2;
  __shared__ uint64_t bar[8], rdy[8];
  __shared__ uint32_t tbase;
  const int G = blockDim.x / 128, g = threadIdx.x / 128, tid = threadIdx.x % 128;
  const uint32_t rank = cta_rank();
  for (int i = threadIdx.x; i < 128 * 128 * 2 + 256 * 128 * 2; i += blockDim.x) sm[i] = 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) { ptx::mbar_init(&bar[i], 1); ptx::mbar_init(&rdy[i], 128); }
    ptx::fence_mbar_init();
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(ptx::smem_u32(&tbase)), "r"(512) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  cluster_sync();
  ptx::tc_fence_after();
  const uint32_t idesc = ptx::idesc_f16(256, n, 0);
  const uint32_t d = tbase + (uint32_t)(g * (512 / G));
  uint32_t phase = 0, rphase = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (handshake && rank == 1) mbar_arrive_remote(&rdy[g], 0);  // peer tile ready
    if (rank == 0 && tid == 0) {
      if (handshake) { ptx::mbar_wait(&rdy[g], rphase); }
      ptx::tc_fence_after();
      for (int ks = 0; ks < ksteps; ++ks) {
        const uint64_t ad = ptx::smem_desc(ptx::smem_u32(A) + ks * 256, 128, 2048, 0);
        const uint64_t bd = ptx::smem_desc(ptx::smem_u32(B) + ks * 256, 128, 2048, 0);
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
            "l"(ad), "l"(bd), "r"(idesc), "r"((uint32_t)(ks > 0))
            : "memory");
      }
      asm volatile(
          "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
              ptx::smem_u32(&bar[g])),
          "h"((uint16_t)3)
          : "memory");
    }
    rphase ^= 1u;
    ptx::mbar_wait(&bar[g], phase);
    phase ^= 1u;
    ptx::tc_fence_after();
    ptx::tc_fence_before();
    ptx::bar_sync(1 + g, 128);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && rank == 0 && blockIdx.x == 0) out[0] = (t1 - t0) / iters;
  ptx::tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (threadIdx.x < 32) {
    ptx::tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(512) : "memory");
  }
}

int main() {
  long long *d, h;
  cudaMalloc(&d, 8);
  const int smem = 128 * 128 * 2 + 256 * 128 * 2 + 2048;
  cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int hs : {0, 1})
    for (int n : {64, 128})
      for (int G : {1, 4})
        for (int ks : {1, 4, 8}) {
          if (G * n > 512) continue;
          k2<<<148, 128 * G, smem>>>(2000, ks, n, hs, d);
          cudaError_t e = cudaDeviceSynchronize();
          cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
          printf("2SM M=256 N=%3d groups=%d ksteps=%d handshake=%d: %5lld cycles/round  %.1f cycles/MMA "
                 "(per SM pair)  (%s)\n",
                 n, G, ks, hs, h, (double)h / (G * ks), cudaGetErrorString(e));
          if (e != cudaSuccess) return 1;
        }
  return 0;
}
