// Microbenchmark: does the way a tcgen05.mma chain is issued set its cost?  The render
// kernel issues from one thread inside `if (tid == 0)`, so ptxas wraps every UTCHMMA in an
// ELECT / R2UR.BROADCAST / BRA.U.ANY loop (divergent code, operands moved to uniform
// registers per instruction).  Style 1 issues from the whole (converged) warp with the
// predicate from `elect.sync` inside the asm, so the descriptors can stay warp-uniform.
// Shape: the render kernel's hidden layer (M = 128, N = 64, 5 K = 16 steps, A from TMEM,
// B in shared memory), 1 or 4 issuing groups per SM, all 148 SMs busy.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_uniform tools/mma_uniform.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2605_18052_b200/csrc/tc_ptx.cuh"

using namespace dmv3d;

__device__ __forceinline__ void mma_ts_elect(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                             uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void commit_elect(uint64_t *bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
          ptx::smem_u32(bar))
      : "memory");
}

// style 0: tid == 0 issues; style 1: warp 0 of the group issues with elect.sync
__global__ void k(int iters, int steps, int style, long long *out) {
  __shared__ __align__(1024) uint8_t B[64 * 80 * 2 * 2];
  __shared__ uint64_t bar[4];
  __shared__ uint32_t tbase;
  const int g = threadIdx.x >> 7, tid = threadIdx.x & 127;
  for (int i = threadIdx.x; i < (int)sizeof(B); i += blockDim.x) B[i] = 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) ptx::mbar_init(&bar[i], 1);
    ptx::fence_mbar_init();
  }
  if (threadIdx.x < 32) ptx::tmem_alloc(&tbase, 512);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tbase + (uint32_t)g * 128u;
  const uint32_t idesc = ptx::idesc_f16(128, 64, 0);
  const uint32_t sB = ptx::smem_u32(B);
  uint32_t phase = 0;
  long long issue = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (style == 0) {
      if (tid == 0) {
        const long long a = clock64();
        ptx::tc_fence_after();
        for (int ks = 0; ks < steps; ++ks) {
          const uint64_t bd = ptx::smem_desc(sB + (ks % 5) * 256, 128, 1280, 0);
          ptx::mma_f16_ts(tmem + 64, tmem + (ks % 4) * 8, bd, idesc, ks > 0);
        }
        ptx::mma_commit(&bar[g]);
        issue += clock64() - a;
      }
    } else {
      if (tid < 32) {
        const long long a = clock64();
        ptx::tc_fence_after();
#pragma unroll 1
        for (int ks = 0; ks < steps; ++ks) {
          const uint64_t bd = ptx::smem_desc(sB + (ks % 5) * 256, 128, 1280, 0);
          mma_ts_elect(tmem + 64, tmem + (ks % 4) * 8, bd, idesc, ks > 0);
        }
        commit_elect(&bar[g]);
        issue += clock64() - a;
      }
    }
    ptx::mbar_wait(&bar[g], phase);
    phase ^= 1u;
    ptx::tc_fence_after();
    ptx::tc_fence_before();
    ptx::bar_sync(1 + g, 128);
  }
  long long t1 = clock64();
  if (tid == 0 && blockIdx.x == 0) {
    out[2 * g] = (t1 - t0) / iters;
    out[2 * g + 1] = issue / iters;
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tbase, 512);
  }
}

int main() {
  long long *d, h[8];
  cudaMalloc(&d, 64);
  printf("groups steps style | round-trip  issue (group 0, cycles per chain)\n");
  for (int groups : {1, 4})
    for (int steps : {1, 2, 5})
      for (int style : {0, 1}) {
        cudaMemset(d, 0, 64);
        k<<<148, 128 * groups>>>(2000, steps, style, d);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
        cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
        printf("%6d %5d %5d | %8lld %8lld\n", groups, steps, style, h[0], h[1]);
      }
  return 0;
}
