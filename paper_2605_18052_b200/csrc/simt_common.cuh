// simt_common.cuh -- fp32 CUDA-core building blocks shared by the SIMT renderer,
// the density grid and the renderer backward: the bilinear triplane gather (a3)
// and the shared MLP with weights resident in shared memory (a4).
#pragma once
#include "common.cuh"
#include "kernels.h"

namespace dmv3d {

// ------------------------------------------------------------ a3: gather
// K = MLP input width; CAT (concat aggregation, row f4): K = 3 C and plane pl
// fills x[pl C, (pl + 1) C), else K = C and the planes are summed (x 1/3: mean).
template <bool BF16, int K, bool CAT = false>
__device__ __forceinline__ void gather_features(const RenderParams &P, const float p[3],
                                                float x[K], int64_t tp_off = 0) {
  constexpr int CP = CAT ? K / 3 : K;
#pragma unroll
  for (int c = 0; c < K; ++c) x[c] = 0.0f;
#pragma unroll
  for (int pl = 0; pl < 3; ++pl) {
    const Cell cell = plane_cell(p, pl, P.R, P.C, P.lo, P.hi, P.inv_ext, P.smode);
    const float w00 = cell.wx0 * cell.wy0, w01 = cell.wx1 * cell.wy0, w10 = cell.wx0 * cell.wy1,
                w11 = cell.wx1 * cell.wy1;
    float *xp = x + (CAT ? pl * CP : 0);
    const int64_t rowC = (int64_t)P.R * P.C;
    if constexpr (BF16) {
      const __nv_bfloat16 *base = reinterpret_cast<const __nv_bfloat16 *>(P.tp) + tp_off + cell.off;
      const uint4 *t00 = reinterpret_cast<const uint4 *>(base);
      const uint4 *t01 = reinterpret_cast<const uint4 *>(base + P.C);
      const uint4 *t10 = reinterpret_cast<const uint4 *>(base + rowC);
      const uint4 *t11 = reinterpret_cast<const uint4 *>(base + rowC + P.C);
#pragma unroll
      for (int q = 0; q < CP / 8; ++q) {
        const uint4 a = __ldg(t00 + q), b = __ldg(t01 + q), c = __ldg(t10 + q), d = __ldg(t11 + q);
        const uint32_t av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
        const uint32_t cv[4] = {c.x, c.y, c.z, c.w}, dv[4] = {d.x, d.y, d.z, d.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          xp[8 * q + 2 * e] += w00 * bf16lo(av[e]) + w01 * bf16lo(bv[e]) + w10 * bf16lo(cv[e]) +
                              w11 * bf16lo(dv[e]);
          xp[8 * q + 2 * e + 1] += w00 * bf16hi(av[e]) + w01 * bf16hi(bv[e]) +
                                  w10 * bf16hi(cv[e]) + w11 * bf16hi(dv[e]);
        }
      }
    } else {
      const float *base = reinterpret_cast<const float *>(P.tp) + tp_off + cell.off;
      const float4 *t00 = reinterpret_cast<const float4 *>(base);
      const float4 *t01 = reinterpret_cast<const float4 *>(base + P.C);
      const float4 *t10 = reinterpret_cast<const float4 *>(base + rowC);
      const float4 *t11 = reinterpret_cast<const float4 *>(base + rowC + P.C);
#pragma unroll
      for (int q = 0; q < CP / 4; ++q) {
        const float4 a = __ldg(t00 + q), b = __ldg(t01 + q), c = __ldg(t10 + q), d = __ldg(t11 + q);
        xp[4 * q + 0] += w00 * a.x + w01 * b.x + w10 * c.x + w11 * d.x;
        xp[4 * q + 1] += w00 * a.y + w01 * b.y + w10 * c.y + w11 * d.y;
        xp[4 * q + 2] += w00 * a.z + w01 * b.z + w10 * c.z + w11 * d.z;
        xp[4 * q + 3] += w00 * a.w + w01 * b.w + w10 * c.w + w11 * d.w;
      }
    }
  }
  if (!CAT && P.agg == 0) {
#pragma unroll
    for (int c = 0; c < K; ++c) x[c] *= (1.0f / 3.0f);
  }
}

// ------------------------------------------------------------ a4: MLP
// Shared-memory layout (fp32): W0 [HD][K], W_l [HD][HD] (l = 1..L-2),
// W_{L-1} [4][HD], then biases b0 [HD], b_l [HD], b_{L-1} [4].
// Pointers are computed, not stored in an indexed array: a runtime layer index into a
// pointer array would place the struct in local memory (one LDL per weight-row access).
template <int K, int HD>
struct MlpSmem {
  float *base;
  int L;
  __device__ __forceinline__ float *W(int l) const {
    return base + (l == 0 ? 0 : K * HD + (l - 1) * HD * HD);
  }
  __device__ __forceinline__ float *B(int l) const {
    return base + K * HD + (L - 2) * HD * HD + 4 * HD + l * HD;
  }
};

template <int K, int HD>
__device__ __forceinline__ int mlp_smem_floats(int L) {
  return HD * K + (L - 2) * HD * HD + 4 * HD + (L - 1) * HD + 4;
}

template <int K, int HD>
__device__ __forceinline__ void fill_weights(const RenderParams &P, const MlpSmem<K, HD> &m,
                                             bool w_bf16) {
  for (int l = 0; l < P.L; ++l) {
    const int in = l == 0 ? K : HD;
    const int out = l == P.L - 1 ? 4 : HD;
    float *dst = m.W(l);
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
__device__ __forceinline__ void mlp_decode(const RenderParams &P, const MlpSmem<K, HD> &m,
                                           const float x[K], float *act, int stride,
                                           float &sigma, float rgb[3]) {
  const int L = P.L;
  // layer 0
  if (L > 1) {
    for (int o = 0; o < HD; ++o) {
      const float *wr = m.W(0) + o * K;
      float acc = m.B(0)[o];
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
      const float *wr = m.W(l) + o * HD;
      float acc = m.B(l)[o];
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
    const float *wr = m.W(L - 1) + o * HD;
    float acc = m.B(L - 1)[o];
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
__device__ __forceinline__ MlpSmem<K, HD> setup_mlp(const RenderParams &P, float *smem, bool w_bf16) {
  MlpSmem<K, HD> m;
  m.base = smem;
  m.L = P.L;
  for (int l = 0; l < P.L; ++l) {
    const int out = l == P.L - 1 ? 4 : HD;
    float *b = m.B(l);
    for (int e = threadIdx.x; e < out; e += blockDim.x) b[e] = __ldg(P.b[l] + e);
  }
  fill_weights<K, HD>(P, m, w_bf16);
  return m;
}

}  // namespace dmv3d
