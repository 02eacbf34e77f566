// Microbenchmark: does shared-memory traffic of the issuing group's other warps slow its
// own tcgen05.mma chain?  One group per SM (all SMs busy): thread 0 issues a 5-step chain
// (M = 128, N = 64, A in TMEM, B in smem) and waits; meanwhile warps 1-3 either idle,
// store to shared memory (st.shared.v4, `work` stores per thread), or issue cp.async
// (L2 -> smem, 16 B each).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_contention tools/mma_contention.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2605_18052_b200/csrc/tc_ptx.cuh"

using namespace dmv3d;

__global__ void k(int iters, int mode, int work, const uint4 *gsrc, long long *out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t *B = sm;              // 10 KB weight-like operand
  uint8_t *S = sm + 16384;      // 64 KB scratch for the traffic
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x;
  for (int i = tid; i < 16384; i += blockDim.x) B[i] = 0;
  if (tid == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
  if (tid < 32) ptx::tmem_alloc(&tbase, 256);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tbase;
  const uint32_t idesc = ptx::idesc_f16(128, 64, 0);
  uint32_t phase = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (tid == 0 && mode < 3) {
      ptx::tc_fence_after();
      for (int ks = 0; ks < 5; ++ks)
        ptx::mma_f16_ts(tmem, tmem + 128 + (ks & 3) * 8, ptx::smem_desc(ptx::smem_u32(B) + ks * 256, 128, 1280, 0),
                        idesc, ks > 0);
      ptx::mma_commit(&bar);
    } else if (tid >= 32) {
      const uint32_t sb = ptx::smem_u32(S);
      if (mode == 1 || mode == 3) {
        for (int w = 0; w < work; ++w)
          ptx::sts128(sb + (uint32_t)(((w * 96 + tid - 32) * 16) & 65535), w, 0u, 0u, 0u);
      } else if (mode == 2 || mode == 4) {
        for (int w = 0; w < work; ++w)
          ptx::cp_async16(sb + (uint32_t)(((w * 96 + tid - 32) * 16) & 65535), gsrc + ((tid + w * 96) & 4095), 16u);
        ptx::cp_async_wait_all();
      }
    }
    if (mode < 3) {
      ptx::mbar_wait(&bar, phase);
      phase ^= 1u;
    }
    ptx::tc_fence_after();
    ptx::tc_fence_before();
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0 && blockIdx.x == 0) out[0] = (t1 - t0) / iters;
  ptx::tc_fence_before();
  __syncthreads();
  if (tid < 32) { ptx::tc_fence_after(); ptx::tmem_dealloc(tbase, 256); }
}

int main() {
  long long *d, h;
  uint4 *g;
  cudaMalloc(&d, 8);
  cudaMalloc(&g, 4096 * 16);
  cudaMemset(g, 0, 4096 * 16);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384 + 65536);
  printf("mode (0 MMA alone, 1 MMA + st.shared, 2 MMA + cp.async, 3 st.shared alone, 4 cp.async alone)  work/thread | cycles per iteration\n");
  for (int mode : {0, 1, 3, 2, 4})
    for (int work : {0, 8, 32, 64}) {
      if (mode == 0 && work > 0) continue;
      k<<<148, 128, 16384 + 65536>>>(2000, mode, work, g, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      printf("%d %4d | %lld\n", mode, work, h);
    }
  // the traffic alone (no MMA) for reference: run with the chain length 0 is not possible
  // here; compare mode 1/2 rows against mode 0 and against the traffic's own issue time
  return 0;
}
