// render_simt.cu -- CUDA-core renderer R(S, c) (+ fused DDIM epilogue).
//
// The fp32 reference-precision engine (DMV3D_ENGINE_SIMT): one warp marches
// one ray in 32-sample chunks, lane = sample.  Per sample: fp32 bilinear
// gather of the three planes (16-byte vector loads, channels-last), the
// shared MLP in fp32 with weights resident in shared memory (broadcast
// reads), then the chunk is composited with a warp-level inclusive scan of
// tau = sigma * delta (transmittance prefix product in log space) and the
// ray stops early once T < term_eps.  Rows a1-a6 of SURVEY.md §8.
#include "common.cuh"
#include "kernels.h"
#include "simt_common.cuh"

namespace dmv3d {

// ------------------------------------------------------ renderer kernel
template <bool BF16, int K, int HD, bool CAT>
__global__ void __launch_bounds__(kSimtThreads)
    render_simt_kernel(const __grid_constant__ RenderParams P, int w_bf16) {
  extern __shared__ __align__(16) float smem[];
  const MlpSmem<K, HD> m = setup_mlp<K, HD>(P, smem, w_bf16 != 0);
  float *act = smem + mlp_smem_floats<K, HD>(P.L);
  act = reinterpret_cast<float *>((reinterpret_cast<uintptr_t>(act) + 15) & ~uintptr_t(15));
  __syncthreads();

  const int lane = threadIdx.x & 31;
  const int64_t warp0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  float *my_act = act + threadIdx.x;
  unsigned long long n_hit = 0, n_samples = 0, n_term = 0, n_rays = 0;

  for (int64_t r = P.ray_begin + warp0; r < P.ray_end; r += nwarps) {
    int v, i, j;
    ray_pixel(r, P.H, P.W, v, i, j);
    if (P.tile_size > 0 && tile_of(v, i, j, P.H, P.W, P.tile_size) % P.tile_count != P.tile_rank)
      continue;  // another rank's tile
    const int act = view_action(P, v);
    if (act != 0) {  // not rendered: nothing, or x_{t-1} = x_t for a kept view
      if (act == 2 && lane < 3) copy_kept(P, v, i, j, lane);
      continue;
    }
    const Ray ray = make_ray(P.intr, P.c2w, v, i, j, P.lo, P.hi);
    if (P.plucker && lane < 6) plucker_write(P.plucker, P.H, P.W, v, i, j, lane, ray);
    n_rays++;
    // batched launch: this view's asset owns the triplane at element offset asset * 3 R R C
    const int64_t tp_off = (int64_t)(v / P.V_asset) * 3 * P.R * P.R * P.C;
    if (!ray.hit) {
      if (lane < 3) ray_epilogue(P, v, i, j, lane, 0.0f, 1.0f);
      continue;
    }
    n_hit++;
    const float delta = sample_delta(ray, P.N);
    float Tc = 1.0f;
    float acc[3] = {0.0f, 0.0f, 0.0f};
    for (int k0 = 0; k0 < P.N; k0 += 32) {
      const int k = k0 + lane;
      const bool valid = k < P.N;
      float sigma = 0.0f, c[3] = {0.0f, 0.0f, 0.0f};
      if (valid) {
        const float u = P.jitter ? jitter_u(P.seed, (uint64_t)r * P.N + k) : 0.5f;
        float p[3];
        sample_p(ray, sample_t(ray, delta, k, u), p);
        float x[K];
        gather_features<BF16, K, CAT>(P, p, x, tp_off);
        mlp_decode<K, HD>(P, m, x, my_act, blockDim.x, sigma, c);
      }
      // a5: front-to-back compositing as a warp prefix sum of optical depth
      const float tau = valid ? sigma * delta : 0.0f;
      float S = tau;
#pragma unroll
      for (int s = 1; s < 32; s <<= 1) {
        const float y = __shfl_up_sync(0xffffffffu, S, s);
        if (lane >= s) S += y;
      }
      const float excl = S - tau;
      const float Tk = Tc * expf(-excl);
      const float w = Tk * (-expm1f(-tau));
#pragma unroll
      for (int ch = 0; ch < 3; ++ch) acc[ch] += w * c[ch];
      const float Stot = __shfl_sync(0xffffffffu, S, 31);
      Tc = Tc * expf(-Stot);
      n_samples += (unsigned long long)min(32, P.N - k0);
      if (Tc < P.term_eps && k0 + 32 < P.N) {
        n_term++;
        break;
      }
    }
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
#pragma unroll
      for (int s = 16; s > 0; s >>= 1) acc[ch] += __shfl_xor_sync(0xffffffffu, acc[ch], s);
    }
    if (lane < 3) ray_epilogue(P, v, i, j, lane, lane == 0 ? acc[0] : (lane == 1 ? acc[1] : acc[2]), Tc);
  }
  if (P.counters && lane == 0) {
    atomicAdd(P.counters + 0, n_hit);
    atomicAdd(P.counters + 1, n_samples);
    atomicAdd(P.counters + 2, n_term);
    atomicAdd(P.counters + 3, n_rays);
  }
}

// --------------------------------------------------------- debug kernels
template <bool BF16, int K, bool CAT>
__global__ void features_kernel(const __grid_constant__ RenderParams P, int64_t n,
                                const float *__restrict__ pts, float *__restrict__ out) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    const float p[3] = {pts[3 * q], pts[3 * q + 1], pts[3 * q + 2]};
    float x[K];
    gather_features<BF16, K, CAT>(P, p, x);
#pragma unroll
    for (int c = 0; c < K; ++c) out[q * K + c] = x[c];
  }
}

template <bool BF16, int K, int HD, bool CAT>
__global__ void __launch_bounds__(kSimtThreads)
    decode_kernel(const __grid_constant__ RenderParams P, int w_bf16, int64_t n,
                  const float *__restrict__ pts, float *__restrict__ out) {
  extern __shared__ __align__(16) float smem[];
  const MlpSmem<K, HD> m = setup_mlp<K, HD>(P, smem, w_bf16 != 0);
  float *act = smem + mlp_smem_floats<K, HD>(P.L);
  act = reinterpret_cast<float *>((reinterpret_cast<uintptr_t>(act) + 15) & ~uintptr_t(15));
  __syncthreads();
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    const float p[3] = {pts[3 * q], pts[3 * q + 1], pts[3 * q + 2]};
    float x[K];
    gather_features<BF16, K, CAT>(P, p, x);
    float sigma, c[3];
    mlp_decode<K, HD>(P, m, x, act + threadIdx.x, blockDim.x, sigma, c);
    out[4 * q] = sigma;
    out[4 * q + 1] = c[0];
    out[4 * q + 2] = c[1];
    out[4 * q + 3] = c[2];
  }
}

// row f3: density grid for marching cubes: G^3 points on the box,
// align-corners, x fastest; sigma [G^3] and optionally rgb [3][G^3]
template <bool BF16, int K, int HD, bool CAT>
__global__ void __launch_bounds__(kSimtThreads)
    density_grid_kernel(const __grid_constant__ RenderParams P, int w_bf16, int G,
                        float *__restrict__ sigma, float *__restrict__ rgb) {
  extern __shared__ __align__(16) float smem[];
  const MlpSmem<K, HD> m = setup_mlp<K, HD>(P, smem, w_bf16 != 0);
  float *act = smem + mlp_smem_floats<K, HD>(P.L);
  act = reinterpret_cast<float *>((reinterpret_cast<uintptr_t>(act) + 15) & ~uintptr_t(15));
  __syncthreads();
  const int64_t n = (int64_t)G * G * G;
  const float gm1 = __int2float_rn(G - 1);
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t id3[3] = {q % G, (q / G) % G, q / ((int64_t)G * G)};
    float p[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const float s = __fdiv_rn(__ll2float_rn(id3[a]), gm1);
      p[a] = __fadd_rn(P.lo[a], __fmul_rn(s, __fsub_rn(P.hi[a], P.lo[a])));
    }
    float x[K];
    gather_features<BF16, K, CAT>(P, p, x);
    float sg, c[3];
    mlp_decode<K, HD>(P, m, x, act + threadIdx.x, blockDim.x, sg, c);
    sigma[q] = sg;
    if (rgb) {
      rgb[q] = c[0];
      rgb[n + q] = c[1];
      rgb[2 * n + q] = c[2];
    }
  }
}

// ------------------------------------------------------------- dispatch
size_t simt_smem_bytes(int K, int HD, int L) {
  size_t floats = (size_t)HD * K + (size_t)(L - 2) * HD * HD + 4 * HD + (size_t)(L - 1) * HD + 4;
  return floats * 4 + 16 + (size_t)HD * kSimtThreads * 4;
}

// (K, HD, CAT): K = MLP input width (3 C for the concat aggregation)
#define DMV3D_SIMT_SHAPES(X) \
  X(4, 16, false)            \
  X(8, 16, false)            \
  X(16, 32, false)           \
  X(32, 64, false)           \
  X(64, 64, false)           \
  X(80, 64, false)           \
  X(12, 16, true)            \
  X(24, 16, true)            \
  X(48, 32, true)            \
  X(96, 64, true)

bool simt_supported(int K, int HD, bool concat) {
#define X(k, h, cat) \
  if (K == k && HD == h && concat == cat) return true;
  DMV3D_SIMT_SHAPES(X)
#undef X
  return false;
}

template <typename Fn>
static cudaError_t launch_cfg(Fn fn, size_t smem, int64_t work_items, int threads, int per_block,
                              cudaStream_t st, int &grid) {
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0, occ = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, smem);
  if (e != cudaSuccess) return e;
  if (occ < 1) occ = 1;
  const int64_t want = (work_items + per_block - 1) / per_block;
  const int64_t cap = (int64_t)sms * occ;
  grid = (int)(want < cap ? (want < 1 ? 1 : want) : cap);
  (void)st;
  return cudaSuccess;
}

cudaError_t launch_render_simt(const RenderParams &P, bool tp_bf16, bool w_bf16,
                               cudaStream_t st) {
  const size_t smem = simt_smem_bytes(P.K, P.HD, P.L);
  const int64_t rays = P.ray_end - P.ray_begin;
  if (rays <= 0) return cudaSuccess;
#define X(k, h, cat)                                                                     \
  if (P.K == k && P.HD == h && (P.agg == 2) == cat) {                                    \
    auto fn = tp_bf16 ? render_simt_kernel<true, k, h, cat> : render_simt_kernel<false, k, h, cat>; \
    int grid = 0;                                                                        \
    cudaError_t e = launch_cfg(fn, smem, rays, kSimtThreads, kSimtThreads / 32, st, grid); \
    if (e != cudaSuccess) return e;                                                      \
    timer_begin(P.timer, st);                                                            \
    fn<<<grid, kSimtThreads, smem, st>>>(P, w_bf16 ? 1 : 0);                             \
    timer_end(P.timer, st);                                                              \
    return cudaGetLastError();                                                           \
  }
  DMV3D_SIMT_SHAPES(X)
#undef X
  return cudaErrorInvalidValue;
}

cudaError_t launch_features(const RenderParams &P, bool tp_bf16, int64_t n, const float *pts,
                            float *out, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int threads = 128;
  const int grid = (int)((n + threads - 1) / threads < 4096 ? (n + threads - 1) / threads : 4096);
#define X(k, cat)                                                                       \
  if (P.C * (cat ? 3 : 1) == k && (P.agg == 2) == cat) {                                \
    auto fn = tp_bf16 ? features_kernel<true, k, cat> : features_kernel<false, k, cat>; \
    fn<<<grid, threads, 0, st>>>(P, n, pts, out);                                       \
    return cudaGetLastError();                                                          \
  }
  X(4, false) X(8, false) X(16, false) X(32, false) X(64, false) X(80, false)
  X(12, true) X(24, true) X(48, true) X(96, true)
#undef X
  return cudaErrorInvalidValue;
}

cudaError_t launch_density_grid(const RenderParams &P, bool tp_bf16, bool w_bf16, int G,
                                float *sigma, float *rgb, cudaStream_t st) {
  const int64_t n = (int64_t)G * G * G;
  if (n <= 0) return cudaSuccess;
  const size_t smem = simt_smem_bytes(P.K, P.HD, P.L);
#define X(k, h, cat)                                                                        \
  if (P.K == k && P.HD == h && (P.agg == 2) == cat) {                                       \
    auto fn = tp_bf16 ? density_grid_kernel<true, k, h, cat> : density_grid_kernel<false, k, h, cat>; \
    int grid = 0;                                                                           \
    cudaError_t e = launch_cfg(fn, smem, n, kSimtThreads, kSimtThreads, st, grid);          \
    if (e != cudaSuccess) return e;                                                         \
    timer_begin(P.timer, st);                                                               \
    fn<<<grid, kSimtThreads, smem, st>>>(P, w_bf16 ? 1 : 0, G, sigma, rgb);                 \
    timer_end(P.timer, st);                                                                 \
    return cudaGetLastError();                                                              \
  }
  DMV3D_SIMT_SHAPES(X)
#undef X
  return cudaErrorInvalidValue;
}

cudaError_t launch_decode(const RenderParams &P, bool tp_bf16, bool w_bf16, int64_t n,
                          const float *pts, float *out, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const size_t smem = simt_smem_bytes(P.K, P.HD, P.L);
#define X(k, h, cat)                                                                    \
  if (P.K == k && P.HD == h && (P.agg == 2) == cat) {                                   \
    auto fn = tp_bf16 ? decode_kernel<true, k, h, cat> : decode_kernel<false, k, h, cat>; \
    int grid = 0;                                                                       \
    cudaError_t e = launch_cfg(fn, smem, n, kSimtThreads, kSimtThreads, st, grid);      \
    if (e != cudaSuccess) return e;                                                     \
    fn<<<grid, kSimtThreads, smem, st>>>(P, w_bf16 ? 1 : 0, n, pts, out);               \
    return cudaGetLastError();                                                          \
  }
  DMV3D_SIMT_SHAPES(X)
#undef X
  return cudaErrorInvalidValue;
}

}  // namespace dmv3d
