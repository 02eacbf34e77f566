// Microbenchmark: MMA-only time of one chunk's MLP sequence per 512 samples on an SM, for
//  (a) the render kernel's shape: 4 groups x 128 samples, each group: blend (SS, 3 K steps,
//      N = 64) -> layer 1 (TS, 5 steps) -> layer 2 (TS, 5 steps) -> head (TS, 2 x 2 steps,
//      N = 16), one round trip (commit + mbarrier wait) per stage;
//  (b) a transposed MLP: 2 groups x 256 samples, each group: 2 blends (SS, 3 steps each,
//      M = 128, N = 64) -> layer 1 (SS, M = 64 outputs, N = 256 samples, 5 steps) ->
//      layer 2 (same) -> head (SS, A MN-major, 2 tiles x 4 steps, N = 16).
// No CUDA-core work: this is the tensor-pipe bound of each design.  All SMs busy.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_mlp_seq tools/mma_mlp_seq.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2605_18052_b200/csrc/tc_ptx.cuh"

using namespace dmv3d;

__device__ __forceinline__ void wait_stage(uint64_t *bar, uint32_t &ph, int g) {
  ptx::mbar_wait(bar, ph);
  ph ^= 1u;
  ptx::tc_fence_after();
  ptx::tc_fence_before();
  ptx::bar_sync(1 + g, 128);
}

__global__ void k(int iters, int design, long long *out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t *A = sm;           // 64 KB operand scratch
  uint8_t *B = sm + 65536;   // 64 KB operand scratch
  __shared__ uint64_t bar[4];
  __shared__ uint32_t tbase;
  const int g = threadIdx.x >> 7, tid = threadIdx.x & 127;
  for (int i = threadIdx.x; i < 131072; i += blockDim.x) sm[i] = 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) ptx::mbar_init(&bar[i], 1);
    ptx::fence_mbar_init();
  }
  if (threadIdx.x < 32) ptx::tmem_alloc(&tbase, 512);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  uint32_t ph = 0;
  const uint32_t a0 = ptx::smem_u32(A), b0 = ptx::smem_u32(B);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (design == 0) {
      const uint32_t tm = tbase + (uint32_t)g * 128u;
      // blend
      if (tid == 0) {
        ptx::tc_fence_after();
        for (int ks = 0; ks < 3; ++ks)
          ptx::mma_f16_ss(tm, ptx::smem_desc(a0 + ks * 256, 128, 2048, 0),
                          ptx::smem_desc(b0 + ks * 2048, 1024, 1024, 2), ptx::idesc_f16(128, 64, 1), ks > 0);
        ptx::mma_commit(&bar[g]);
      }
      wait_stage(&bar[g], ph, g);
      for (int l = 0; l < 2; ++l) {
        if (tid == 0) {
          ptx::tc_fence_after();
          for (int ks = 0; ks < 5; ++ks)
            ptx::mma_f16_ts(tm, tm + 64 + (ks & 3) * 8, ptx::smem_desc(b0 + ks * 256, 128, 1280, 0),
                            ptx::idesc_f16(128, 64, 0), ks > 0);
          ptx::mma_commit(&bar[g]);
        }
        wait_stage(&bar[g], ph, g);
      }
      if (tid == 0) {
        ptx::tc_fence_after();
        for (int ks = 0; ks < 2; ++ks)
          for (int hx = 0; hx < 2; ++hx)
            ptx::mma_f16_ts(tm + (hx ? 112u : 0u), tm + 64 + (2 * hx + ks) * 8,
                            ptx::smem_desc(b0 + ks * 256, 128, 1280, 0), ptx::idesc_f16(128, 16, 0), ks > 0);
        ptx::mma_commit(&bar[g]);
      }
      wait_stage(&bar[g], ph, g);
    } else {
      const uint32_t tm = tbase + (uint32_t)g * 256u;
      if (tid == 0) {  // two blends (two 128-sample halves) into columns 0 and 64
        ptx::tc_fence_after();
        for (int h = 0; h < 2; ++h)
          for (int ks = 0; ks < 3; ++ks)
            ptx::mma_f16_ss(tm + h * 64, ptx::smem_desc(a0 + h * 32768 + ks * 256, 128, 2048, 0),
                            ptx::smem_desc(b0 + ks * 2048, 1024, 1024, 2), ptx::idesc_f16(128, 64, 1), ks > 0);
        ptx::mma_commit(&bar[g]);
      }
      wait_stage(&bar[g], ph, g);
      for (int l = 0; l < 2; ++l) {
        if (tid == 0) {  // D^T [64 x 256] = W [64 x 80] . H^T [80 x 256]
          ptx::tc_fence_after();
          for (int ks = 0; ks < 5; ++ks)
            ptx::mma_f16_ss(tm, ptx::smem_desc(a0 + ks * 256, 128, 1280, 0),
                            ptx::smem_desc(b0 + ks * 256, 128, 2048, 0), ptx::idesc_f16(64, 256, 0), ks > 0);
          ptx::mma_commit(&bar[g]);
        }
        wait_stage(&bar[g], ph, g);
      }
      if (tid == 0) {  // head, both halves: A = H^T read MN-major
        ptx::tc_fence_after();
        for (int h = 0; h < 2; ++h)
          for (int ks = 0; ks < 4; ++ks)
            ptx::mma_f16_ss(tm + h * 16, ptx::smem_desc(b0 + h * 16384 + ks * 2048, 1024, 128, 0),
                            ptx::smem_desc(a0 + ks * 256, 128, 1280, 0),
                            ptx::idesc_f16(128, 16, 0) | (1u << 15), ks > 0);
        ptx::mma_commit(&bar[g]);
      }
      wait_stage(&bar[g], ph, g);
    }
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
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072 + 1024);
  for (int design : {0, 1}) {
    const int groups = design == 0 ? 4 : 2;
    cudaMemset(d, 0, 32);
    k<<<148, 128 * groups, 131072 + 1024>>>(1000, design, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
    printf("design %s: %d groups, %lld cycles per iteration (= 512 samples per SM)\n",
           design == 0 ? "current (4 x 128 rows)" : "transposed MLP (2 x 256 samples)", groups, h[0]);
  }
  return 0;
}
