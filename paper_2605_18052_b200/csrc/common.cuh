// common.cuh -- device-side building blocks shared by the libdmv3d kernels.
//
// Geometry (rows a1-a3 of SURVEY.md §8) is computed with explicit IEEE
// round-to-nearest intrinsics, one rounding per operation and no FMA
// contraction, so the integer/geometry outputs are bit-identical to any
// implementation that follows the same operation order (DESIGN.md
// "Bit-exact geometry").  Everything after the texel indices is ordinary
// fp32 (or bf16 tensor-core) arithmetic.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace dmv3d {

constexpr int kMaxLayers = 8;
constexpr int kMaxPeers = 7;  // the other GPUs of an 8-GPU node

// All per-launch parameters; passed by value as a __grid_constant__.
struct RenderParams {
  // camera set C; a batched launch renders `V / V_asset` assets of
  // V_asset views each (global view v = asset * V_asset + local view)
  int32_t V, H, W;
  int32_t V_asset;
  const float *intr;  // [V][4]
  const float *c2w;   // [V][3][4]
  // triplane S
  int32_t R, C;
  const void *tp;  // [3][R][R][C]
  float lo[3], hi[3];
  float inv_ext[3];  // 1/(hi-lo) if a power of two, else 0 (see texel_coord)
  int32_t smode;     // texel addressing: 0 align-corners/clamp, 1 half-pixel/zeros (f4)
  int32_t tp_fp8;    // storage FP8 E4M3 (value = tp_scale * e4m3; TC engine only, f4)
  float tp_scale;
  // shared MLP
  int32_t L, K, HD;
  const void *w[kMaxLayers];
  const float *b[kMaxLayers];
  int32_t act;
  float dshift, weps;
  // ray marching
  int32_t N, agg, jitter;
  uint64_t seed;
  float bg[3];
  float term_eps;
  int64_t ray_begin, ray_end;
  // outputs
  float *rgb;    // [V][3][H][W] or null
  float *alpha;  // [V][H][W] or null
  // fused DDIM epilogue, views [0, ddim_views)
  int32_t ddim_views;
  uint64_t keep_bits;
  const float *x_t, *z;
  float *x_prev;
  float x0_scale, x0_shift;
  float sqrt_ab_t, inv_sqrt_1m_ab_t, sqrt_ab_p, c_eps, sigma_t;
  int32_t ddim_only;  // fused step without rgb/alpha: views >= ddim_views are not rendered
  int32_t skip_kept;  // kept views (keep_bits) are not rendered: x_{t-1} = x_t copied
  uint64_t noise_seed;  // z == null && sigma_t != 0: in-kernel noise (row f4)
  unsigned long long *counters;
  // caller-owned scratch (tensor-core engine: patch counter + projected triplane)
  void *ws;
  size_t ws_bytes;
  // optional host-side launch timer (dmv3d_timer*): events around the render kernel
  void *timer;
  // optional Plucker ray map output [V][6][H][W] (row f2), written during a1
  float *plucker;
  // P2P copies of every output value (view-sharded multi-GPU step): peer buffers laid
  // out like rgb / alpha / x_prev
  int32_t npeers;
  float *peer_rgb[kMaxPeers], *peer_alpha[kMaxPeers], *peer_xp[kMaxPeers];
  // interleaved ray tiles: tile_size > 0 keeps only the pixels of tiles
  // tau = (v ceil(H/T) + i/T) ceil(W/T) + j/T with tau mod tile_count == tile_rank
  int32_t tile_size, tile_rank, tile_count;
  // host-pipelined step: G in the workspace is current (skip K0, only reset the counter)
  int32_t reuse_g;
  // density grid mode of the tensor-core engine (row f3): G^3 points, x fastest
  int32_t grid_res;
  float *grid_sigma, *grid_rgb;
};

// ---------------------------------------------------------------- ray tiles (§8e)
__host__ __device__ inline int64_t tile_of(int v, int i, int j, int H, int W, int T) {
  const int64_t th = (H + T - 1) / T, tw = (W + T - 1) / T;
  return ((int64_t)v * th + i / T) * tw + j / T;
}
// tiles of views [v_lo, v_hi] owned by `rank`: the first id and how many
__host__ __device__ inline void owned_tiles(int v_lo, int v_hi, int H, int W, int T, int rank,
                                            int count, int64_t &first, int64_t &n) {
  const int64_t per_view = (int64_t)((H + T - 1) / T) * ((W + T - 1) / T);
  const int64_t t0 = (int64_t)v_lo * per_view, t1 = (int64_t)(v_hi + 1) * per_view;
  first = t0 + (((int64_t)rank - t0) % count + count) % count;
  n = first < t1 ? (t1 - first + count - 1) / count : 0;
}

// ---------------------------------------------------------------- a1: rays
// Pinhole camera, pixel centre at +1/2, OpenCV axes, unit direction.
struct Ray {
  float o[3], d[3];
  float t_near, t_far;
  bool hit;
};

__device__ __forceinline__ void ray_pixel(int64_t r, int H, int W, int &v, int &i, int &j) {
  const int64_t HW = (int64_t)H * W;
  const int64_t vv = r / HW;
  const int64_t rem = r - vv * HW;
  const int64_t ii = rem / W;
  v = (int)vv;
  i = (int)ii;
  j = (int)(rem - ii * W);
}

__device__ __forceinline__ Ray make_ray(const float *__restrict__ intr,
                                        const float *__restrict__ c2w, int v, int i, int j,
                                        const float lo[3], const float hi[3]) {
  Ray ray;
  const float *K = intr + 4 * v;
  const float *M = c2w + 12 * v;
  const float xc = __fdiv_rn(__fsub_rn(__fadd_rn(__int2float_rn(j), 0.5f), __ldg(K + 2)),
                             __ldg(K + 0));
  const float yc = __fdiv_rn(__fsub_rn(__fadd_rn(__int2float_rn(i), 0.5f), __ldg(K + 3)),
                             __ldg(K + 1));
  float dw[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const float s = __fadd_rn(__fmul_rn(__ldg(M + 4 * a + 0), xc), __fmul_rn(__ldg(M + 4 * a + 1), yc));
    dw[a] = __fadd_rn(s, __ldg(M + 4 * a + 2));
  }
  const float nn = __fadd_rn(__fadd_rn(__fmul_rn(dw[0], dw[0]), __fmul_rn(dw[1], dw[1])),
                             __fmul_rn(dw[2], dw[2]));
  const float n = __fsqrt_rn(nn);
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    ray.d[a] = __fdiv_rn(dw[a], n);
    ray.o[a] = __ldg(M + 4 * a + 3);
  }
  // a2: slab test against [lo, hi] (reading A9)
  bool ok = true;
  float tmin[3], tmax[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    if (ray.d[a] == 0.0f) {
      ok = ok && !(ray.o[a] < lo[a] || ray.o[a] > hi[a]);
      tmin[a] = -INFINITY;
      tmax[a] = INFINITY;
    } else {
      const float t0 = __fdiv_rn(__fsub_rn(lo[a], ray.o[a]), ray.d[a]);
      const float t1 = __fdiv_rn(__fsub_rn(hi[a], ray.o[a]), ray.d[a]);
      tmin[a] = fminf(t0, t1);
      tmax[a] = fmaxf(t0, t1);
    }
  }
  const float tn = fmaxf(fmaxf(fmaxf(tmin[0], tmin[1]), tmin[2]), 0.0f);
  const float tf = fminf(fminf(tmax[0], tmax[1]), tmax[2]);
  ray.hit = ok && (tf > tn);
  ray.t_near = ray.hit ? tn : 0.0f;
  ray.t_far = ray.hit ? tf : 0.0f;
  return ray;
}

// ------------------------------------------------------------- a2: samples
// Reading A10: optional stratified jitter, splitmix64 finaliser on the
// sample id (portable counter-based generator).
__device__ __forceinline__ float jitter_u(uint64_t seed, uint64_t sample_id) {
  uint64_t z = seed + (sample_id + 1ull) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z = z ^ (z >> 31);
  return __fmul_rn(__uint2float_rn((uint32_t)(z >> 40)), 1.0f / 16777216.0f);
}

// Row f4: in-kernel DDIM noise for element e of x_t, Box-Muller on two 24-bit
// splitmix64 uniforms (u1 in (0,1], u2 in [0,1)).
__device__ __forceinline__ uint64_t splitmix_at(uint64_t seed, uint64_t ctr) {
  uint64_t z = seed + ctr * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ float ddim_noise(uint64_t seed, uint64_t e) {
  const float u1 = (float)((splitmix_at(seed, 2 * e + 1) >> 40) + 1) * (1.0f / 16777216.0f);
  const float u2 = (float)(splitmix_at(seed, 2 * e + 2) >> 40) * (1.0f / 16777216.0f);
  return sqrtf(-2.0f * logf(u1)) * cospif(2.0f * u2);
}

__device__ __forceinline__ float sample_delta(const Ray &ray, int N) {
  return __fdiv_rn(__fsub_rn(ray.t_far, ray.t_near), __int2float_rn(N));
}

__device__ __forceinline__ float sample_t(const Ray &ray, float delta, int k, float u) {
  return __fadd_rn(ray.t_near, __fmul_rn(__fadd_rn(__int2float_rn(k), u), delta));
}

__device__ __forceinline__ void sample_p(const Ray &ray, float t, float p[3]) {
#pragma unroll
  for (int a = 0; a < 3; ++a) p[a] = __fadd_rn(ray.o[a], __fmul_rn(t, ray.d[a]));
}

// ------------------------------------------------------------ a3: texels
// Reading A3: align-corners, clamped; i0 in [0, R-2], f in [0, 1].
// `inv` = 1/(hi - lo) when hi - lo is a power of two (then x/(hi-lo) and
// x*inv are the same correctly rounded value), else 0 (IEEE division).
__device__ __forceinline__ void texel_coord(float q, float lo, float hi, float inv, int R,
                                            int &i0, float &f) {
  const float num = __fsub_rn(q, lo);
  const float s = (inv != 0.0f) ? __fmul_rn(num, inv) : __fdiv_rn(num, __fsub_rn(hi, lo));
  float px = __fmul_rn(s, __int2float_rn(R - 1));
  px = fminf(fmaxf(px, 0.0f), __int2float_rn(R - 1));
  int ix = __float2int_rd(px);
  ix = min(ix, R - 2);
  i0 = ix;
  f = __fsub_rn(px, __int2float_rn(ix));
}

// Row f4: half-pixel texel centres, (i + 1/2)/R of the box; the unclamped lower
// index i0 = floor(s R - 1/2) lies in [-1, R-1] for points in the box.
__device__ __forceinline__ void texel_coord_hp(float q, float lo, float hi, float inv, int R,
                                               int &i0, float &f) {
  const float num = __fsub_rn(q, lo);
  const float s = (inv != 0.0f) ? __fmul_rn(num, inv) : __fdiv_rn(num, __fsub_rn(hi, lo));
  const float px = __fsub_rn(__fmul_rn(s, __int2float_rn(R)), 0.5f);
  const int ix = __float2int_rd(px);
  i0 = ix;
  f = __fsub_rn(px, __int2float_rn(ix));
}

// One axis of a bilinear cell in either addressing mode: the cell base i0 in
// [0, R-2] and the weights of texels i0 and i0 + 1.  Half-pixel corners that
// fall outside the plane get weight zero (zero padding), so every mode reads
// the same in-range 2x2 cell.
__device__ __forceinline__ void texel_axis(float q, float lo, float hi, float inv, int R,
                                           int mode, int &i0, float &w0, float &w1) {
  int ix;
  float f;
  if (mode == 0) {
    texel_coord(q, lo, hi, inv, R, ix, f);
    i0 = ix;
    w0 = 1.0f - f;
    w1 = f;
    return;
  }
  texel_coord_hp(q, lo, hi, inv, R, ix, f);
  const float g = 1.0f - f;
  if (ix < 0) {  // only texel ix + 1 = 0 can be inside
    i0 = 0;
    w0 = ix == -1 ? f : 0.0f;
    w1 = 0.0f;
  } else if (ix > R - 2) {  // only texel ix = R - 1 can be inside
    i0 = R - 2;
    w0 = 0.0f;
    w1 = ix == R - 1 ? g : 0.0f;
  } else {
    i0 = ix;
    w0 = g;
    w1 = f;
  }
}

// Plane (a, b) for planes XY, XZ, YZ (reading A2).
__device__ __forceinline__ int plane_axis_a(int pl) { return pl == 2 ? 1 : 0; }
__device__ __forceinline__ int plane_axis_b(int pl) { return pl == 0 ? 1 : 2; }

// One plane's bilinear cell: element offset of texel (iy, ix) and the per-axis
// weights (corner (y, x) weighs wy[y] * wx[x]).
struct Cell {
  int64_t off;  // element offset of corner (iy, ix) of plane pl
  float wx0, wx1, wy0, wy1;
};

__device__ __forceinline__ Cell plane_cell(const float p[3], int pl, int R, int C,
                                           const float lo[3], const float hi[3],
                                           const float inv[3], int mode) {
  const int a = plane_axis_a(pl), b = plane_axis_b(pl);
  int ix, iy;
  Cell c;
  texel_axis(p[a], lo[a], hi[a], inv[a], R, mode, ix, c.wx0, c.wx1);
  texel_axis(p[b], lo[b], hi[b], inv[b], R, mode, iy, c.wy0, c.wy1);
  c.off = (((int64_t)pl * R + iy) * R + ix) * C;
  return c;
}

// ---------------------------------------------------------------- helpers
__device__ __forceinline__ float softplus_f(float x) {
  return log1pf(expf(-fabsf(x))) + fmaxf(x, 0.0f);
}
__device__ __forceinline__ float sigmoid_f(float x) { return 1.0f / (1.0f + expf(-x)); }
__device__ __forceinline__ float hidden_act_f(int kind, float x) {
  if (kind == 1) return x * sigmoid_f(x);
  if (kind == 2) return softplus_f(x);
  return fmaxf(x, 0.0f);
}

__device__ __forceinline__ float bf16lo(uint32_t u) { return __uint_as_float(u << 16); }
__device__ __forceinline__ float bf16hi(uint32_t u) { return __uint_as_float(u & 0xffff0000u); }

// Plucker coordinates r = (o x d, d), component c in 0..5; each
// moment component is two rounded products and one rounded difference.
__device__ __forceinline__ float plucker_component(const Ray &ray, int c) {
  if (c >= 3) return ray.d[c - 3];
  const int a = (c + 1) % 3, b = (c + 2) % 3;
  return __fsub_rn(__fmul_rn(ray.o[a], ray.d[b]), __fmul_rn(ray.o[b], ray.d[a]));
}

__device__ __forceinline__ void plucker_write(float *out, int H, int W, int v, int i, int j,
                                              int c, const Ray &ray) {
  const int64_t HW = (int64_t)H * W;
  out[((int64_t)v * 6 + c) * HW + (int64_t)i * W + j] = plucker_component(ray, c);
}

// NVLink stores of one output value into the peers' buffers (out of line: keeps the
// renderers' register allocation unchanged when no peers are given)
static __device__ __noinline__ void peer_store_rgb(const RenderParams &P, int64_t irgb, int64_t ia, int ch,
                                            float rgb, float a) {
  for (int k = 0; k < P.npeers; ++k) {
    if (P.peer_rgb[k]) P.peer_rgb[k][irgb] = rgb;
    if (ch == 0 && P.peer_alpha[k]) P.peer_alpha[k][ia] = a;
  }
}
static __device__ __noinline__ void peer_store_xp(const RenderParams &P, int64_t idx, float xp) {
  for (int k = 0; k < P.npeers; ++k)
    if (P.peer_xp[k]) P.peer_xp[k][idx] = xp;
}

__device__ __forceinline__ bool kept_view(const RenderParams &P, int vl) {
  return vl < 64 && ((P.keep_bits >> vl) & 1ull);
}

// What a fused step does with the rays of global view v: 0 = render, 1 = nothing
// (ddim_only: a view >= ddim_views whose rgb/alpha nobody asked for), 2 = copy x_t into
// x_{t-1} without rendering (skip_kept: a kept conditioning view).
__device__ __forceinline__ int view_action(const RenderParams &P, int v) {
  if (!P.ddim_only && !P.skip_kept) return 0;
  const int vl = v % P.V_asset;
  if (P.ddim_only && vl >= P.ddim_views) return 1;
  if (P.skip_kept && vl < P.ddim_views && kept_view(P, vl)) return 2;
  return 0;
}
// x_{t-1} = x_t for channel ch of pixel (i, j) of a kept view (view_action == 2)
__device__ __forceinline__ void copy_kept(const RenderParams &P, int v, int i, int j, int ch) {
  const int64_t HW = (int64_t)P.H * P.W;
  const int a = v / P.V_asset, vl = v - a * P.V_asset;
  const int64_t idx = (((int64_t)a * P.ddim_views + vl) * 3 + ch) * HW + (int64_t)i * P.W + j;
  const float xt = __ldg(P.x_t + idx);
  P.x_prev[idx] = xt;
  if (P.npeers) peer_store_xp(P, idx, xt);
}

// Per-ray epilogue: write rgb/alpha and, for DDIM views, x_{t-1}
// (readings A15, A18-A20).  `ch` selects the channel this
// thread writes (0..2); channel 0's thread also writes alpha.  Batched launches:
// view v is local view v % V_asset of asset v / V_asset; x_t / z / x_{t-1} are
// [assets][ddim_views][3][H][W].
__device__ __forceinline__ void ray_epilogue(const RenderParams &P, int v, int i, int j, int ch,
                                             float c_val, float T) {
  const int64_t HW = (int64_t)P.H * P.W;
  const int64_t pix = (int64_t)i * P.W + j;
  const float out = c_val + T * P.bg[ch];
  const int64_t irgb = ((int64_t)v * 3 + ch) * HW + pix, ia = (int64_t)v * HW + pix;
  if (P.rgb) P.rgb[irgb] = out;
  if (ch == 0 && P.alpha) P.alpha[ia] = 1.0f - T;
  if (P.npeers) peer_store_rgb(P, irgb, ia, ch, out, 1.0f - T);
  const int a = v / P.V_asset, vl = v - a * P.V_asset;
  if (vl < P.ddim_views) {
    const int64_t idx = (((int64_t)a * P.ddim_views + vl) * 3 + ch) * HW + pix;
    const float xt = __ldg(P.x_t + idx);
    float xp;
    if (kept_view(P, vl)) {
      xp = xt;
    } else {
      const float x0 = P.x0_scale * out + P.x0_shift;
      const float eps = (xt - P.sqrt_ab_t * x0) * P.inv_sqrt_1m_ab_t;
      xp = P.sqrt_ab_p * x0 + P.c_eps * eps;
      if (P.sigma_t != 0.0f)
        xp += P.sigma_t * (P.z ? __ldg(P.z + idx) : ddim_noise(P.noise_seed, (uint64_t)idx));
    }
    P.x_prev[idx] = xp;
    if (P.npeers) peer_store_xp(P, idx, xp);
  }
}

}  // namespace dmv3d
