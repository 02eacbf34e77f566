// Microbenchmark: cost of a dependent tcgen05.mma accumulation chain vs the shared-
// memory operand layout (SWIZZLE_NONE interleaved vs SWIZZLE_128B K-major), 1 CTA,
// one issuing thread.  Operand contents are zero: only timing is measured.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_swizzle tools/mma_swizzle.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2605_18052_b200/csrc/tc_ptx.cuh"
using namespace dmv3d;

// layout 0: K-major interleaved core matrices, LBO = 128 (K direction), SBO = 2048
// (8-row groups of a 128-row x 128-K tile); a K = 16 step advances 256 B.
// layout 2: K-major SWIZZLE_128B, 64 K per 128-B row, SBO = 1024 (8-row atoms); a
// K = 16 step advances 32 B inside the atom, every 4 steps the next 64-K slab.
__device__ __forceinline__ uint64_t desc(uint32_t base, int layout, int ks, int rows) {
  if (layout == 0) return ptx::smem_desc(base + ks * 256, 128, 2048, 0);
  const uint32_t slab = (uint32_t)(ks >> 2) * (uint32_t)rows * 128u;
  return ptx::smem_desc(base + slab + (ks & 3) * 32, 16, 1024, 2);
}

__global__ void k(int iters, int ksteps, int n, int layout, int chains, long long *out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
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
        for (int c = 0; c < chains; ++c)
          ptx::mma_f16_ss(tbase + c * n, desc(ptx::smem_u32(A), layout, ks, 128),
                          desc(ptx::smem_u32(B), layout, ks, 256), idesc, ks > 0);
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
  const int smem = 128 * 128 * 2 + 256 * 128 * 2 + 2048;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int layout : {0})
    for (int n : {16, 64, 128, 256})
      for (int chains : {1, 2, 4, 8})
        for (int ks : {1, 8}) {
          if (chains * n > 512) continue;
          k<<<1, 128, smem>>>(2000, ks, n, layout, chains, d);
          cudaError_t e = cudaDeviceSynchronize();
          cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
          printf("layout=%d N=%3d chains=%d ksteps=%d : %5lld cycles/round trip  (%s)\n", layout, n,
                 chains, ks, h, cudaGetErrorString(e));
        }
  return 0;
}
