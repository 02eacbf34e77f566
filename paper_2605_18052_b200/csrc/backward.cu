// backward.cu -- renderer backward: gradients of
// L = <g_rgb, rgb> + <g_alpha, alpha> w.r.t. the triplane and the shared MLP,
// the "differentiable volume rendering" that L_recon trains through
// (PAPER.md:47-55, :71).  fp32 CUDA cores, ReLU hidden layers.
//
// One warp per ray, lane = sample in 32-sample chunks, two passes:
//   1. forward: composite the ray to get C = sum_k w_k c_k + T_N bg and T_N;
//   2. forward again storing every layer's input in shared memory, then per
//      sample dC/dtau_k = T_{k+1} c_k - R_k with R_k = C - sum_{j<=k} w_j c_j
//      (a warp prefix sum), dA/dtau_k = T_N, dC/dc_k = w_k; back through the
//      MLP; the feature gradient is scattered to the 12 bilinear corners with
//      fp32 atomics; weight gradients are outer products summed over the
//      warp's 32 samples in registers (lane = output row) and added with one
//      atomic per weight per chunk.
// Accumulates into caller-zeroed fp32 buffers (atomic order => results are
// deterministic only up to fp32 rounding).
#include "common.cuh"
#include "kernels.h"
#include "simt_common.cuh"

namespace dmv3d {

constexpr int kBwThreads = 128;

template <int K, int HD>
__device__ __forceinline__ void mlp_forward_store(const RenderParams &P, const MlpSmem<K, HD> &m,
                                                  float *col, int stride, float o4[4]) {
  // col rows: [0, K) = h0, [K + (l-1) HD, K + l HD) = h_l (l >= 1, post-ReLU)
  const int L = P.L;
  for (int l = 0; l < L - 1; ++l) {
    const int in = l == 0 ? K : HD;
    const float *hin = col + (l == 0 ? 0 : (K + (l - 1) * HD)) * stride;
    float *hout = col + (K + l * HD) * stride;
    for (int o = 0; o < HD; ++o) {
      const float *wr = m.W(l) + o * in;
      float acc = m.B(l)[o];
      for (int i = 0; i < in; i += 4) {
        const float4 w4 = *reinterpret_cast<const float4 *>(wr + i);
        acc += w4.x * hin[i * stride] + w4.y * hin[(i + 1) * stride] + w4.z * hin[(i + 2) * stride] +
               w4.w * hin[(i + 3) * stride];
      }
      hout[o * stride] = fmaxf(acc, 0.0f);
    }
  }
  const float *h = col + (L == 1 ? 0 : (K + (L - 2) * HD)) * stride;
  const int in = L == 1 ? K : HD;
#pragma unroll
  for (int o = 0; o < 4; ++o) {
    const float *wr = m.W(L - 1) + o * in;
    float acc = m.B(L - 1)[o];
    for (int i = 0; i < in; ++i) acc += wr[i] * h[i * stride];
    o4[o] = acc;
  }
}

template <bool BF16, int K, int HD, bool CAT>
__global__ void __launch_bounds__(kBwThreads, 1)
    render_backward_kernel(const __grid_constant__ RenderParams P,
                           const __grid_constant__ GradParams Gp, int w_bf16) {
  extern __shared__ __align__(16) float smem[];
  const MlpSmem<K, HD> m = setup_mlp<K, HD>(P, smem, w_bf16 != 0);
  float *scratch = smem + mlp_smem_floats<K, HD>(P.L);
  scratch = reinterpret_cast<float *>((reinterpret_cast<uintptr_t>(scratch) + 15) & ~uintptr_t(15));
  const int L = P.L;
  const int rows = K + (L - 1) * HD;
  constexpr int kDs = HD + 4;  // padded delta row: a lane's LDS.128 hits distinct banks
  float *dstage = scratch + rows * kBwThreads;  // [warps][32 samples][kDs]
  __syncthreads();

  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  float *col = scratch + threadIdx.x;               // this lane's column (stride 128)
  float *wcol = scratch + wib * 32;                  // the warp's 32 columns
  float *dst = dstage + wib * 32 * kDs;              // [32][kDs]
  const int64_t warp0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const float scale = (!CAT && P.agg == 0) ? (1.0f / 3.0f) : 1.0f;
  constexpr int CP = CAT ? K / 3 : K;  // channels per plane
  const int64_t HWp = (int64_t)P.H * P.W;

  for (int64_t r = P.ray_begin + warp0; r < P.ray_end; r += nwarps) {
    int v, i, j;
    ray_pixel(r, P.H, P.W, v, i, j);
    const Ray ray = make_ray(P.intr, P.c2w, v, i, j, P.lo, P.hi);
    if (!ray.hit) continue;
    const int64_t pix = (int64_t)i * P.W + j;
    float g[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) g[c] = __ldg(Gp.g_rgb + ((int64_t)v * 3 + c) * HWp + pix);
    const float gA = Gp.g_alpha ? __ldg(Gp.g_alpha + (int64_t)v * HWp + pix) : 0.0f;
    const float delta = sample_delta(ray, P.N);

    // ---- pass 1: C and T_N (or the caller's forward render)
    float Tc = 1.0f, acc[3] = {0.f, 0.f, 0.f};
    const bool have_fwd = Gp.fwd_rgb != nullptr;
    int kstop = P.N;  // the chunk after which the ray stopped (pass 1)
    if (have_fwd) {
      Tc = 1.0f - __ldg(Gp.fwd_alpha + (int64_t)v * HWp + pix);
#pragma unroll
      for (int c = 0; c < 3; ++c)  // C = acc + Tc bg below (acc summed over the warp)
        acc[c] = lane == 0 ? __ldg(Gp.fwd_rgb + ((int64_t)v * 3 + c) * HWp + pix) - Tc * P.bg[c] : 0.0f;
    }
    for (int k0 = 0; k0 < (have_fwd ? 0 : P.N); k0 += 32) {
      const int k = k0 + lane;
      const bool valid = k < P.N;
      float sigma = 0.0f, c[3] = {0.f, 0.f, 0.f};
      if (valid) {
        const float u = P.jitter ? jitter_u(P.seed, (uint64_t)r * P.N + k) : 0.5f;
        float p[3];
        sample_p(ray, sample_t(ray, delta, k, u), p);
        float x[K];
        gather_features<BF16, K, CAT>(P, p, x);
        mlp_decode<K, HD>(P, m, x, col, kBwThreads, sigma, c);
      }
      const float tau = valid ? sigma * delta : 0.0f;
      float S = tau;
#pragma unroll
      for (int s = 1; s < 32; s <<= 1) {
        const float y = __shfl_up_sync(0xffffffffu, S, s);
        if (lane >= s) S += y;
      }
      const float w = Tc * expf(-(S - tau)) * (-expm1f(-tau));
#pragma unroll
      for (int c2 = 0; c2 < 3; ++c2) acc[c2] += w * c[c2];
      Tc *= expf(-__shfl_sync(0xffffffffu, S, 31));
      if (P.term_eps > 0.0f && Tc < P.term_eps) {  // the forward's early termination
        kstop = k0;
        break;
      }
    }
    float Ctot[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
#pragma unroll
      for (int s = 16; s > 0; s >>= 1) acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], s);
      Ctot[c] = acc[c] + Tc * P.bg[c];
    }
    const float TN = Tc;

    // ---- pass 2: forward with stored activations, then backward
    Tc = 1.0f;
    float Pc[3] = {0.f, 0.f, 0.f};
    for (int k0 = 0; k0 < P.N; k0 += 32) {
      const int k = k0 + lane;
      const bool valid = k < P.N;
      float p[3] = {0.f, 0.f, 0.f};
      float o4[4] = {0.f, 0.f, 0.f, 0.f};
      if (valid) {
        const float u = P.jitter ? jitter_u(P.seed, (uint64_t)r * P.N + k) : 0.5f;
        sample_p(ray, sample_t(ray, delta, k, u), p);
        float x[K];
        gather_features<BF16, K, CAT>(P, p, x);
#pragma unroll
        for (int c = 0; c < K; ++c) col[c * kBwThreads] = x[c];
        mlp_forward_store<K, HD>(P, m, col, kBwThreads, o4);
      } else {
        for (int rr = 0; rr < rows; ++rr) col[rr * kBwThreads] = 0.0f;
      }
      const float z0 = o4[0] + P.dshift;
      const float sigma = valid ? (log1pf(expf(-fabsf(z0))) + fmaxf(z0, 0.0f)) : 0.0f;
      float c[3], sg[3];
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        sg[q] = sigmoid_f(o4[1 + q]);
        c[q] = valid ? sg[q] * (1.0f + 2.0f * P.weps) - P.weps : 0.0f;
      }
      const float tau = valid ? sigma * delta : 0.0f;
      float S = tau;
#pragma unroll
      for (int s = 1; s < 32; s <<= 1) {
        const float y = __shfl_up_sync(0xffffffffu, S, s);
        if (lane >= s) S += y;
      }
      const float Tk = Tc * expf(-(S - tau));
      const float w = Tk * (-expm1f(-tau));
      const float Tk1 = Tk * expf(-tau);
      float R[3], tot[3];
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        float sc = w * c[q];
#pragma unroll
        for (int s = 1; s < 32; s <<= 1) {
          const float y = __shfl_up_sync(0xffffffffu, sc, s);
          if (lane >= s) sc += y;
        }
        R[q] = Ctot[q] - (Pc[q] + sc);
        tot[q] = __shfl_sync(0xffffffffu, sc, 31);
      }
      float dtau = gA * TN;
#pragma unroll
      for (int q = 0; q < 3; ++q) dtau += g[q] * (Tk1 * c[q] - R[q]);
      // ---- the head's delta (dL/d o, o = sigma / rgb pre-activations) -> this lane's
      //      staged row; all deltas live in shared memory (no per-thread arrays)
      float *myd = dst + lane * kDs;
      {
        float4 d4 = make_float4(0.f, 0.f, 0.f, 0.f);
        if (valid) {
          const float cs = w * (1.0f + 2.0f * P.weps);
          d4 = make_float4(dtau * delta * sigmoid_f(z0), g[0] * cs * sg[0] * (1.0f - sg[0]),
                           g[1] * cs * sg[1] * (1.0f - sg[1]), g[2] * cs * sg[2] * (1.0f - sg[2]));
        }
        *reinterpret_cast<float4 *>(myd) = d4;
      }
      // ---- back through the MLP, layer L-1 .. 0
      for (int l = L - 1; l >= 0; --l) {
        const int in = l == 0 ? K : HD;
        const int out = l == L - 1 ? 4 : HD;
        const int hrow = l == 0 ? 0 : K + (l - 1) * HD;
        __syncwarp();  // every lane's delta row is staged
        // dW_l += d (x) h_l, db_l += d: lanes own output rows q, summing the warp's 32 samples
        for (int q = lane; q < out; q += 32) {
          float dq[32];
          float bsum = 0.0f;
#pragma unroll
          for (int s = 0; s < 32; ++s) {
            dq[s] = dst[s * kDs + q];
            bsum += dq[s];
          }
          if (bsum != 0.0f) atomicAdd(Gp.db[l] + q, bsum);
          for (int ii = 0; ii < in; ++ii) {
            const float *hr = wcol + (hrow + ii) * kBwThreads;
            float sum = 0.0f;
#pragma unroll
            for (int s = 0; s < 32; ++s) sum += dq[s] * hr[s];
            if (sum != 0.0f) atomicAdd(Gp.dW[l] + (size_t)q * in + ii, sum);
          }
        }
        __syncwarp();  // h_l is consumed: it may be overwritten by dh
        // dh = W_l^T d (lane = sample), 16 inputs at a time: 4-wide broadcast weight loads
        // against the lane's own delta row; ReLU-masked by h_l > 0 for l > 0, written over h_l
        const float *W = m.W(l);
        for (int i0 = 0; i0 < in; i0 += 16) {
          float acc[16];
#pragma unroll
          for (int t = 0; t < 16; ++t) acc[t] = 0.0f;
          for (int q = 0; q < out; q += 4) {
            const float4 d4 = *reinterpret_cast<const float4 *>(myd + q);
            const float dv[4] = {d4.x, d4.y, d4.z, d4.w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const float *wr = W + (q + j) * in + i0;
#pragma unroll
              for (int t = 0; t < 16; t += 4) {
                if (i0 + t < in) {
                  const float4 w4 = *reinterpret_cast<const float4 *>(wr + t);
                  acc[t] += w4.x * dv[j];
                  acc[t + 1] += w4.y * dv[j];
                  acc[t + 2] += w4.z * dv[j];
                  acc[t + 3] += w4.w * dv[j];
                }
              }
            }
          }
#pragma unroll
          for (int t = 0; t < 16; ++t) {
            if (i0 + t < in) {
              float *c = col + (hrow + i0 + t) * kBwThreads;
              *c = (l == 0 || *c > 0.0f) ? acc[t] : 0.0f;
            }
          }
        }
        if (l > 0) {
          // the next delta (layer l-1's outputs) = the masked dh just written
          for (int q = 0; q < HD; q += 4)
            *reinterpret_cast<float4 *>(myd + q) =
                make_float4(col[(hrow + q) * kBwThreads], col[(hrow + q + 1) * kBwThreads],
                            col[(hrow + q + 2) * kBwThreads], col[(hrow + q + 3) * kBwThreads]);
        } else {
          // dL/dh0 (rows [0, K) of this lane's column) -> the 12 bilinear corners of the
          // three planes, x the aggregation scale
          const int64_t rowC = (int64_t)P.R * P.C;
          float wcs[3][4];
          int64_t offs[3];
#pragma unroll
          for (int pl = 0; pl < 3; ++pl) {
            const Cell cell = plane_cell(p, pl, P.R, P.C, P.lo, P.hi, P.inv_ext, P.smode);
            const float sc = valid ? scale : 0.0f;
            wcs[pl][0] = cell.wx0 * cell.wy0 * sc;
            wcs[pl][1] = cell.wx1 * cell.wy0 * sc;
            wcs[pl][2] = cell.wx0 * cell.wy1 * sc;
            wcs[pl][3] = cell.wx1 * cell.wy1 * sc;
            offs[pl] = cell.off;
          }
          constexpr int NCH = (K + 31) / 32;
          if (32 * NCH <= (L - 1) * HD) {
            // Lanes switch from samples to channels, so each RED covers 32 consecutive
            // channels of one texel instead of 32 scattered texels: dh0 goes through a
            // skewed sample-major scratch in the warp's dead hidden-activation rows, each
            // sample's cells and corner weights through its (dead) delta row.
            uint32_t *cr = reinterpret_cast<uint32_t *>(myd);
#pragma unroll
            for (int pl = 0; pl < 3; ++pl) {
              cr[pl * 6] = (uint32_t)((uint64_t)offs[pl] & 0xffffffffu);
              cr[pl * 6 + 1] = (uint32_t)((uint64_t)offs[pl] >> 32);
#pragma unroll
              for (int e = 0; e < 4; ++e) cr[pl * 6 + 2 + e] = __float_as_uint(wcs[pl][e]);
            }
            float *tsc = wcol + K * kBwThreads;
            for (int c = 0; c < K; ++c)
              tsc[(lane * NCH + (c >> 5)) * kBwThreads + ((c + lane) & 31)] = valid ? col[c * kBwThreads] : 0.0f;
            __syncwarp();
            for (int s2 = 0; s2 < 32; ++s2) {
              const uint32_t *cs = reinterpret_cast<const uint32_t *>(dst + s2 * kDs);
#pragma unroll
              for (int pl = 0; pl < 3; ++pl) {
                const float w0 = __uint_as_float(cs[pl * 6 + 2]), w1 = __uint_as_float(cs[pl * 6 + 3]);
                const float w2 = __uint_as_float(cs[pl * 6 + 4]), w3 = __uint_as_float(cs[pl * 6 + 5]);
                if (w0 == 0.0f && w1 == 0.0f && w2 == 0.0f && w3 == 0.0f) continue;  // warp-uniform
                const int64_t off = (int64_t)(((uint64_t)cs[pl * 6 + 1] << 32) | cs[pl * 6]);
                const int x0 = CAT ? pl * CP : 0;
                for (int k0 = 0; k0 < CP; k0 += 32) {
                  const int cc = k0 + lane;
                  if (cc < CP) {
                    const int c = x0 + cc;
                    const float v = tsc[(s2 * NCH + (c >> 5)) * kBwThreads + ((c + s2) & 31)];
                    if (w0 != 0.0f) atomicAdd(Gp.dF + off + cc, w0 * v);
                    if (w1 != 0.0f) atomicAdd(Gp.dF + off + P.C + cc, w1 * v);
                    if (w2 != 0.0f) atomicAdd(Gp.dF + off + rowC + cc, w2 * v);
                    if (w3 != 0.0f) atomicAdd(Gp.dF + off + rowC + P.C + cc, w3 * v);
                  }
                }
              }
            }
          } else if (valid) {
#pragma unroll
            for (int pl = 0; pl < 3; ++pl) {
              const int64_t off[4] = {offs[pl], offs[pl] + P.C, offs[pl] + rowC, offs[pl] + rowC + P.C};
              const int x0 = CAT ? pl * CP : 0;  // this plane's columns of h0
              for (int cc = 0; cc < CP; ++cc) {
                const float dh = col[(x0 + cc) * kBwThreads];
#pragma unroll
                for (int e = 0; e < 4; ++e)
                  if (wcs[pl][e] != 0.0f) atomicAdd(Gp.dF + off[e] + cc, wcs[pl][e] * dh);
              }
            }
          }
        }
      }
      __syncwarp();
      Tc *= expf(-__shfl_sync(0xffffffffu, S, 31));
#pragma unroll
      for (int q = 0; q < 3; ++q) Pc[q] += tot[q];
      if (k0 == kstop || (have_fwd && P.term_eps > 0.0f && Tc < P.term_eps)) break;
    }
  }
}

template <typename Fn>
static cudaError_t bw_launch(Fn fn, size_t smem, int64_t rays, cudaStream_t st, const RenderParams &P,
                            const GradParams &Gp, int w_bf16) {
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t grid = (rays + 3) / 4;
  if (grid > sms) grid = sms;
  timer_begin(P.timer, st);
  fn<<<(int)grid, kBwThreads, smem, st>>>(P, Gp, w_bf16);
  timer_end(P.timer, st);
  return cudaGetLastError();
}

size_t backward_smem_bytes(int K, int HD, int L) {
  const size_t mlp = (size_t)HD * K + (size_t)(L - 2) * HD * HD + 4 * HD + (size_t)(L - 1) * HD + 4;
  return (mlp + 4 + (size_t)(K + (L - 1) * HD) * kBwThreads + (size_t)4 * 32 * (HD + 4)) * 4;
}

#define DMV3D_BW_SHAPES(X) \
  X(4, 16, false)          \
  X(8, 16, false)          \
  X(16, 32, false)         \
  X(32, 64, false)         \
  X(80, 64, false)         \
  X(12, 16, true)          \
  X(24, 16, true)          \
  X(48, 32, true)

bool backward_supported(int K, int HD, int L, bool concat) {
  if (backward_smem_bytes(K, HD, L) > 232448) return false;
#define X(k, h, cat) \
  if (K == k && HD == h && concat == cat) return true;
  DMV3D_BW_SHAPES(X)
#undef X
  return false;
}

cudaError_t launch_render_backward(const RenderParams &P, const GradParams &Gp, bool tp_bf16,
                                   bool w_bf16, cudaStream_t st) {
  const int64_t rays = P.ray_end - P.ray_begin;
  if (rays <= 0) return cudaSuccess;
  const size_t smem = backward_smem_bytes(P.K, P.HD, P.L);
#define X(k, h, cat)                                                                                  \
  if (P.K == k && P.HD == h && (P.agg == 2) == cat)                                                   \
    return tp_bf16 ? bw_launch(render_backward_kernel<true, k, h, cat>, smem, rays, st, P, Gp, w_bf16) \
                   : bw_launch(render_backward_kernel<false, k, h, cat>, smem, rays, st, P, Gp, w_bf16);
  DMV3D_BW_SHAPES(X)
#undef X
  return cudaErrorInvalidValue;
}

}  // namespace dmv3d
