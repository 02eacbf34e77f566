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

namespace dmv3d {

// ------------------------------------------------------------ a3: gather
template <bool BF16, int K>
__device__ __forceinline__ void gather_features(const RenderParams &P, const float p[3],
                                                float x[K]) {
#pragma unroll
  for (int c = 0; c < K; ++c) x[c] = 0.0f;
#pragma unroll
  for (int pl = 0; pl < 3; ++pl) {
    const Cell cell = plane_cell(p, pl, P.R, P.C, P.lo, P.hi, P.inv_ext);
    const float gx = 1.0f - cell.fx, gy = 1.0f - cell.fy;
    const float w00 = gx * gy, w01 = cell.fx * gy, w10 = gx * cell.fy, w11 = cell.fx * cell.fy;
    const int64_t rowC = (int64_t)P.R * P.C;
    if constexpr (BF16) {
      const __nv_bfloat16 *base = reinterpret_cast<const __nv_bfloat16 *>(P.tp) + cell.off;
      const uint4 *t00 = reinterpret_cast<const uint4 *>(base);
      const uint4 *t01 = reinterpret_cast<const uint4 *>(base + P.C);
      const uint4 *t10 = reinterpret_cast<const uint4 *>(base + rowC);
      const uint4 *t11 = reinterpret_cast<const uint4 *>(base + rowC + P.C);
#pragma unroll
      for (int q = 0; q < K / 8; ++q) {
        const uint4 a = __ldg(t00 + q), b = __ldg(t01 + q), c = __ldg(t10 + q), d = __ldg(t11 + q);
        const uint32_t av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
        const uint32_t cv[4] = {c.x, c.y, c.z, c.w}, dv[4] = {d.x, d.y, d.z, d.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          x[8 * q + 2 * e] += w00 * bf16lo(av[e]) + w01 * bf16lo(bv[e]) + w10 * bf16lo(cv[e]) +
                              w11 * bf16lo(dv[e]);
          x[8 * q + 2 * e + 1] += w00 * bf16hi(av[e]) + w01 * bf16hi(bv[e]) +
                                  w10 * bf16hi(cv[e]) + w11 * bf16hi(dv[e]);
        }
      }
    } else {
      const float *base = reinterpret_cast<const float *>(P.tp) + cell.off;
      const float4 *t00 = reinterpret_cast<const float4 *>(base);
      const float4 *t01 = reinterpret_cast<const float4 *>(base + P.C);
      const float4 *t10 = reinterpret_cast<const float4 *>(base + rowC);
      const float4 *t11 = reinterpret_cast<const float4 *>(base + rowC + P.C);
#pragma unroll
      for (int q = 0; q < K / 4; ++q) {
        const float4 a = __ldg(t00 + q), b = __ldg(t01 + q), c = __ldg(t10 + q), d = __ldg(t11 + q);
        x[4 * q + 0] += w00 * a.x + w01 * b.x + w10 * c.x + w11 * d.x;
        x[4 * q + 1] += w00 * a.y + w01 * b.y + w10 * c.y + w11 * d.y;
        x[4 * q + 2] += w00 * a.z + w01 * b.z + w10 * c.z + w11 * d.z;
        x[4 * q + 3] += w00 * a.w + w01 * b.w + w10 * c.w + w11 * d.w;
      }
    }
  }
  if (P.agg == 0) {
#pragma unroll
    for (int c = 0; c < K; ++c) x[c] *= (1.0f / 3.0f);
  }
}

// ------------------------------------------------------------ a4: MLP
// Shared-memory layout (fp32): W0 [HD][K], W_l [HD][HD] (l = 1..L-2),
// W_{L-1} [4][HD], then biases b0 [HD], b_l [HD], b_{L-1} [4].
struct MlpSmem {
  const float *W[kMaxLayers];
  const float *B[kMaxLayers];
};

template <int K, int HD>
__device__ __forceinline__ int mlp_smem_floats(int L) {
  return HD * K + (L - 2) * HD * HD + 4 * HD + (L - 1) * HD + 4;
}

template <int K, int HD>
__device__ __forceinline__ void fill_weights(const RenderParams &P, const MlpSmem &m,
                                             bool w_bf16) {
  for (int l = 0; l < P.L; ++l) {
    const int in = l == 0 ? K : HD;
    const int out = l == P.L - 1 ? 4 : HD;
    float *dst = const_cast<float *>(m.W[l]);
    const int n = in * out;
    if (w_bf16) {
      const __nv_bfloat16 *src = reinterpret_cast<const __nv_bfloat16 *>(P.w[l]);
      for (int e = threadIdx.x; e < n; e += blockDim.x) dst[e] = __bfloat162float(src[e]);
    } else {
      const float *src = reinterpret_cast<const float *>(P.w[l]);
      for (int e = threadIdx.x; e < n; e += blockDim.x) dst[e] = __ldg(src + e);
    }
  }
}

// h0 [K] in registers -> (sigma, rgb).  `act` is this thread's column of a
// [HD][blockDim] fp32 scratch (stride blockDim), conflict-free.
template <int K, int HD>
__device__ __forceinline__ void mlp_decode(const RenderParams &P, const MlpSmem &m,
                                           const float x[K], float *act, int stride,
                                           float &sigma, float rgb[3]) {
  const int L = P.L;
  // layer 0
  if (L > 1) {
    for (int o = 0; o < HD; ++o) {
      const float *wr = m.W[0] + o * K;
      float acc = m.B[0][o];
#pragma unroll
      for (int i = 0; i < K; i += 4) {
        const float4 w4 = *reinterpret_cast<const float4 *>(wr + i);
        acc += w4.x * x[i] + w4.y * x[i + 1] + w4.z * x[i + 2] + w4.w * x[i + 3];
      }
      act[o * stride] = hidden_act_f(P.act, acc);
    }
  }
  // hidden layers 1..L-2
  for (int l = 1; l < L - 1; ++l) {
    float h[HD];
#pragma unroll
    for (int i = 0; i < HD; ++i) h[i] = act[i * stride];
    for (int o = 0; o < HD; ++o) {
      const float *wr = m.W[l] + o * HD;
      float acc = m.B[l][o];
#pragma unroll
      for (int i = 0; i < HD; i += 4) {
        const float4 w4 = *reinterpret_cast<const float4 *>(wr + i);
        acc += w4.x * h[i] + w4.y * h[i + 1] + w4.z * h[i + 2] + w4.w * h[i + 3];
      }
      act[o * stride] = hidden_act_f(P.act, acc);
    }
  }
  // head HD -> 4
  float h[HD];
#pragma unroll
  for (int i = 0; i < HD; ++i) h[i] = act[i * stride];
  float o4[4];
#pragma unroll
  for (int o = 0; o < 4; ++o) {
    const float *wr = m.W[L - 1] + o * HD;
    float acc = m.B[L - 1][o];
#pragma unroll
    for (int i = 0; i < HD; i += 4) {
      const float4 w4 = *reinterpret_cast<const float4 *>(wr + i);
      acc += w4.x * h[i] + w4.y * h[i + 1] + w4.z * h[i + 2] + w4.w * h[i + 3];
    }
    o4[o] = acc;
  }
  sigma = softplus_f(o4[0] + P.dshift);
#pragma unroll
  for (int c = 0; c < 3; ++c) rgb[c] = sigmoid_f(o4[1 + c]) * (1.0f + 2.0f * P.weps) - P.weps;
}

template <int K, int HD>
__device__ __forceinline__ MlpSmem setup_mlp(const RenderParams &P, float *smem, bool w_bf16) {
  MlpSmem m;
  float *cur = smem;
  for (int l = 0; l < P.L; ++l) {
    const int in = l == 0 ? K : HD;
    const int out = l == P.L - 1 ? 4 : HD;
    m.W[l] = cur;
    cur += in * out;
  }
  for (int l = 0; l < P.L; ++l) {
    const int out = l == P.L - 1 ? 4 : HD;
    m.B[l] = cur;
    for (int e = threadIdx.x; e < out; e += blockDim.x) cur[e] = __ldg(P.b[l] + e);
    cur += out;
  }
  fill_weights<K, HD>(P, m, w_bf16);
  return m;
}

// ------------------------------------------------------ renderer kernel
template <bool BF16, int K, int HD>
__global__ void __launch_bounds__(kSimtThreads)
    render_simt_kernel(const __grid_constant__ RenderParams P, int w_bf16) {
  extern __shared__ __align__(16) float smem[];
  const MlpSmem m = setup_mlp<K, HD>(P, smem, w_bf16 != 0);
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
    const Ray ray = make_ray(P.intr, P.c2w, v, i, j, P.lo, P.hi);
    if (P.plucker && lane < 6) plucker_write(P.plucker, P.H, P.W, v, i, j, lane, ray);
    n_rays++;
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
        gather_features<BF16, K>(P, p, x);
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
template <bool BF16, int K>
__global__ void features_kernel(const __grid_constant__ RenderParams P, int64_t n,
                                const float *__restrict__ pts, float *__restrict__ out) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    const float p[3] = {pts[3 * q], pts[3 * q + 1], pts[3 * q + 2]};
    float x[K];
    gather_features<BF16, K>(P, p, x);
#pragma unroll
    for (int c = 0; c < K; ++c) out[q * K + c] = x[c];
  }
}

template <bool BF16, int K, int HD>
__global__ void __launch_bounds__(kSimtThreads)
    decode_kernel(const __grid_constant__ RenderParams P, int w_bf16, int64_t n,
                  const float *__restrict__ pts, float *__restrict__ out) {
  extern __shared__ __align__(16) float smem[];
  const MlpSmem m = setup_mlp<K, HD>(P, smem, w_bf16 != 0);
  float *act = smem + mlp_smem_floats<K, HD>(P.L);
  act = reinterpret_cast<float *>((reinterpret_cast<uintptr_t>(act) + 15) & ~uintptr_t(15));
  __syncthreads();
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    const float p[3] = {pts[3 * q], pts[3 * q + 1], pts[3 * q + 2]};
    float x[K];
    gather_features<BF16, K>(P, p, x);
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
template <bool BF16, int K, int HD>
__global__ void __launch_bounds__(kSimtThreads)
    density_grid_kernel(const __grid_constant__ RenderParams P, int w_bf16, int G,
                        float *__restrict__ sigma, float *__restrict__ rgb) {
  extern __shared__ __align__(16) float smem[];
  const MlpSmem m = setup_mlp<K, HD>(P, smem, w_bf16 != 0);
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
    gather_features<BF16, K>(P, p, x);
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

#define DMV3D_SIMT_SHAPES(X) \
  X(4, 16)                   \
  X(8, 16)                   \
  X(16, 32)                  \
  X(32, 64)                  \
  X(64, 64)                  \
  X(80, 64)

bool simt_supported(int K, int HD) {
#define X(k, h) \
  if (K == k && HD == h) return true;
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
#define X(k, h)                                                                          \
  if (P.K == k && P.HD == h) {                                                           \
    auto fn = tp_bf16 ? render_simt_kernel<true, k, h> : render_simt_kernel<false, k, h>; \
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
#define X(k, h)                                                               \
  if (P.C == k) {                                                             \
    auto fn = tp_bf16 ? features_kernel<true, k> : features_kernel<false, k>; \
    fn<<<grid, threads, 0, st>>>(P, n, pts, out);                             \
    return cudaGetLastError();                                                \
  }
  X(4, 0) X(8, 0) X(16, 0) X(32, 0) X(64, 0) X(80, 0)
#undef X
  return cudaErrorInvalidValue;
}

cudaError_t launch_density_grid(const RenderParams &P, bool tp_bf16, bool w_bf16, int G,
                                float *sigma, float *rgb, cudaStream_t st) {
  const int64_t n = (int64_t)G * G * G;
  if (n <= 0) return cudaSuccess;
  const size_t smem = simt_smem_bytes(P.K, P.HD, P.L);
#define X(k, h)                                                                             \
  if (P.K == k && P.HD == h) {                                                              \
    auto fn = tp_bf16 ? density_grid_kernel<true, k, h> : density_grid_kernel<false, k, h>; \
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
#define X(k, h)                                                                         \
  if (P.K == k && P.HD == h) {                                                          \
    auto fn = tp_bf16 ? decode_kernel<true, k, h> : decode_kernel<false, k, h>;         \
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
