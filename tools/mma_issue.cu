// Microbenchmark: how long the issuing thread spends in a tcgen05.mma chain (issue loop +
// commit) versus the chain's round trip (issue -> commit -> mbarrier wait), for the
// render kernel's layer shape (M = 128, N = 64, K = 16 per step, A from TMEM, B in smem),
// with the K steps as one dependent chain or split over independent accumulators, and
// with 1..4 issuing groups per SM (all 148 SMs busy).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_issue tools/mma_issue.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2605_18052_b200/csrc/tc_ptx.cuh"

using namespace dmv3d;

// groups x 128 threads; group g owns TMEM columns [g*160, g*160+160): the A operand at
// +0..31 (K = 64 as 4 steps of 8 columns), accumulator D0 at +32, D1 at +96 (64 columns
// each).  `steps` K steps are spread round robin over `chains` accumulators.
__global__ void k(int iters, int steps, int chains, int split_threads, int n, long long *out) {
  __shared__ __align__(1024) uint8_t B[64 * 80 * 2 * 2];
  __shared__ uint64_t bar[4];
  __shared__ uint32_t tbase;
  const int g = threadIdx.x >> 7, tid = threadIdx.x & 127;
  const int ng = blockDim.x >> 7;
  for (int i = threadIdx.x; i < (int)sizeof(B); i += blockDim.x) B[i] = 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) ptx::mbar_init(&bar[i], split_threads ? chains : 1);
    ptx::fence_mbar_init();
  }
  if (threadIdx.x < 32) ptx::tmem_alloc(&tbase, 512);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tbase + (uint32_t)g * 160u;
  const uint32_t idesc = ptx::idesc_f16(128, n, 0);
  uint32_t phase = 0;
  long long issue = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    // split_threads: chain c is issued by lane 0 of warp c of the group (every issuing
    // thread commits; the mbarrier expects `chains` arrivals)
    const int me = split_threads ? (tid >> 5) : 0;
    if ((tid & 31) == 0 && (split_threads ? me < chains : tid == 0)) {
      const long long a = clock64();
      ptx::tc_fence_after();
      for (int ks = 0; ks < steps; ++ks) {
        const int c = ks % chains;
        if (split_threads && c != me) continue;
        const uint64_t bd = ptx::smem_desc(ptx::smem_u32(B) + (ks % 5) * 256, 128, 1280, 0);
        ptx::mma_f16_ts(tmem + (c ? 96u : 32u), tmem + (ks % 4) * 8, bd, idesc, ks >= chains);
      }
      ptx::mma_commit(&bar[g]);
      if (me == 0) issue += clock64() - a;
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
  (void)ng;
}

int main() {
  long long *d, h[8];
  cudaMalloc(&d, 64);
  printf("grid groups  n steps chains threads | round-trip  issue (group 0)\n");
  for (int grid : {148})
    for (int groups : {1, 3})
      for (int n : {64, 32})
        for (int split : {0, 1})
          for (int chains : {1, 2})
            for (int steps : {2, 4, 5}) {
              if (chains > steps || (split && chains == 1)) continue;
              cudaMemset(d, 0, 64);
              k<<<grid, 128 * groups>>>(2000, steps, chains, split, n, d);
              cudaError_t e = cudaDeviceSynchronize();
              if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
              cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
              printf("%4d %6d %3d %5d %6d %7d | %8lld %8lld\n", grid, groups, n, steps, chains, split, h[0], h[1]);
            }
  return 0;
}
