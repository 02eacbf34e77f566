// Microbenchmark: can the issuing group (all 4 warps, including the issuing thread's warp)
// do CUDA-core work while its own tcgen05.mma chain runs?  One group per SM, all SMs:
//   mode 0: work, then issue the 5-step chain, wait      (serial)
//   mode 1: issue, work, wait                            (work in the chain's shadow)
//   mode 2: issue, work with a group barrier in the middle, wait
//   mode 3: issue, shared-memory stores, wait
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_shadow tools/mma_shadow.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2605_18052_b200/csrc/tc_ptx.cuh"

using namespace dmv3d;

__device__ __forceinline__ float alu_work(float x, int n) {
#pragma unroll 1
  for (int i = 0; i < n; ++i) x = fmaf(x, 1.0001f, 0.5f) * 0.999f;  // dependent chain
  return x;
}

__global__ void k(int iters, int mode, int work, float *sink, long long *out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t *B = sm, *S = sm + 16384;
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
  float x = (float)tid;
  auto issue = [&]() {
    if (tid == 0) {
      ptx::tc_fence_after();
      for (int ks = 0; ks < 5; ++ks)
        ptx::mma_f16_ts(tmem, tmem + 128 + (ks & 3) * 8, ptx::smem_desc(ptx::smem_u32(B) + ks * 256, 128, 1280, 0),
                        idesc, ks > 0);
      ptx::mma_commit(&bar);
    }
  };
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (mode == 0) { x = alu_work(x, work); issue(); }
    else if (mode == 1) { issue(); x = alu_work(x, work); }
    else if (mode == 2) { issue(); x = alu_work(x, work / 2); ptx::bar_sync(1, 128); x = alu_work(x, work / 2); }
    else {
      issue();
      const uint32_t sb = ptx::smem_u32(S);
      for (int w = 0; w < work / 8; ++w) ptx::sts128(sb + (uint32_t)(((w * 128 + tid) * 16) & 65535), w, 0u, 0u, 0u);
    }
    ptx::mbar_wait(&bar, phase);
    phase ^= 1u;
    ptx::tc_fence_after();
    ptx::tc_fence_before();
    ptx::bar_sync(1, 128);
  }
  long long t1 = clock64();
  if (tid == 0 && blockIdx.x == 0) out[0] = (t1 - t0) / iters;
  sink[blockIdx.x * blockDim.x + tid] = x;
  ptx::tc_fence_before();
  __syncthreads();
  if (tid < 32) { ptx::tc_fence_after(); ptx::tmem_dealloc(tbase, 256); }
}

int main() {
  long long *d, h;
  float *sink;
  cudaMalloc(&d, 8);
  cudaMalloc(&sink, 148 * 128 * 4);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384 + 65536);
  printf("mode (0 work;issue  1 issue;work  2 issue;work+barrier  3 issue;smem stores)  work | cycles/iter\n");
  for (int work : {0, 50, 100, 200})
    for (int mode : {0, 1, 2, 3}) {
      k<<<148, 128, 16384 + 65536>>>(2000, mode, work, sink, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      printf("%d %4d | %lld\n", mode, work, h);
    }
  return 0;
}
