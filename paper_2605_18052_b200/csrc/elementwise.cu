// elementwise.cu -- standalone DDIM step (row a6) and the stage-level debug
// kernels for rows a1-a3 (bit-exact geometry dumps).
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace dmv3d {

// ------------------------------------------------------------------ a6
// x0 = s*rgb + b; eps = (x_t - sqrt(ab_t) x0) / sqrt(1 - ab_t);
// x_{t-1} = sqrt(ab_p) x0 + c_eps eps + sigma_t z
__device__ __forceinline__ float ddim_one(const DdimCoef &c, float xt, float rgb, float z) {
  const float x0 = c.x0_scale * rgb + c.x0_shift;
  const float eps = (xt - c.sqrt_ab_t * x0) * c.inv_sqrt_1m_ab_t;
  float xp = c.sqrt_ab_p * x0 + c.c_eps * eps;
  if (c.sigma_t != 0.0f) xp += c.sigma_t * z;
  return xp;
}

// HBM-bound: 16-byte loads/stores, grid = multiple of the SM count.
__global__ void ddim_kernel(const __grid_constant__ DdimCoef c, int64_t per_view, int64_t n4,
                            const float4 *__restrict__ x_t, const float4 *__restrict__ x0,
                            const float4 *__restrict__ z, float4 *__restrict__ out) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n4;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int v = (int)((q * 4) / per_view);
    const float4 xt = __ldg(x_t + q);
    if (v < 64 && ((c.keep_bits >> v) & 1ull)) {  // keep_mask covers <= 64 views
      out[q] = xt;
      continue;
    }
    const float4 r = __ldg(x0 + q);
    float4 zz = make_float4(0.f, 0.f, 0.f, 0.f);
    if (c.sigma_t != 0.0f) {
      if (z) {
        zz = __ldg(z + q);
      } else {
        zz.x = ddim_noise(c.noise_seed, 4 * q);
        zz.y = ddim_noise(c.noise_seed, 4 * q + 1);
        zz.z = ddim_noise(c.noise_seed, 4 * q + 2);
        zz.w = ddim_noise(c.noise_seed, 4 * q + 3);
      }
    }
    float4 o;
    o.x = ddim_one(c, xt.x, r.x, zz.x);
    o.y = ddim_one(c, xt.y, r.y, zz.y);
    o.z = ddim_one(c, xt.z, r.z, zz.z);
    o.w = ddim_one(c, xt.w, r.w, zz.w);
    out[q] = o;
  }
}

__global__ void ddim_kernel_scalar(const __grid_constant__ DdimCoef c, int64_t per_view,
                                   int64_t n, const float *__restrict__ x_t,
                                   const float *__restrict__ x0, const float *__restrict__ z,
                                   float *__restrict__ out) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int v = (int)(q / per_view);
    const float xt = x_t[q];
    const float zq = c.sigma_t == 0.0f ? 0.0f : (z ? z[q] : ddim_noise(c.noise_seed, (uint64_t)q));
    out[q] = (v < 64 && ((c.keep_bits >> v) & 1ull)) ? xt : ddim_one(c, xt, x0[q], zq);
  }
}

static int sm_count() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

cudaError_t launch_ddim(const DdimCoef &c, int V, int H, int W, const float *x_t,
                        const float *x0_rgb, const float *z, const uint8_t *, float *x_prev,
                        cudaStream_t st) {
  const int64_t per_view = (int64_t)3 * H * W;
  const int64_t n = per_view * V;
  if (n == 0) return cudaSuccess;
  const int threads = 256;
  if (per_view % 4 == 0) {
    const int64_t n4 = n / 4;
    int64_t grid = (n4 + threads - 1) / threads;
    const int64_t cap = (int64_t)sm_count() * 8;
    if (grid > cap) grid = cap;
    ddim_kernel<<<(int)grid, threads, 0, st>>>(c, per_view, n4,
                                               reinterpret_cast<const float4 *>(x_t),
                                               reinterpret_cast<const float4 *>(x0_rgb),
                                               reinterpret_cast<const float4 *>(z),
                                               reinterpret_cast<float4 *>(x_prev));
  } else {
    int64_t grid = (n + threads - 1) / threads;
    const int64_t cap = (int64_t)sm_count() * 8;
    if (grid > cap) grid = cap;
    ddim_kernel_scalar<<<(int)grid, threads, 0, st>>>(c, per_view, n, x_t, x0_rgb, z, x_prev);
  }
  return cudaGetLastError();
}

// ------------------------------------------------------- a1-a3 debug dumps
__global__ void ray_geometry_kernel(const __grid_constant__ RenderParams P, float *o_d,
                                    float *tn_tf, uint8_t *hit) {
  const int64_t n = P.ray_end - P.ray_begin;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    int v, i, j;
    ray_pixel(P.ray_begin + q, P.H, P.W, v, i, j);
    const Ray ray = make_ray(P.intr, P.c2w, v, i, j, P.lo, P.hi);
    if (o_d) {
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        o_d[6 * q + a] = ray.o[a];
        o_d[6 * q + 3 + a] = ray.d[a];
      }
    }
    if (tn_tf) {
      tn_tf[2 * q] = ray.t_near;
      tn_tf[2 * q + 1] = ray.t_far;
    }
    if (hit) hit[q] = ray.hit ? 1 : 0;
  }
}

__global__ void sample_points_kernel(const __grid_constant__ RenderParams P, float *t_k,
                                     float *points, int32_t *texel, float *frac) {
  const int64_t n = (P.ray_end - P.ray_begin) * P.N;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t rr = q / P.N;
    const int k = (int)(q - rr * P.N);
    const int64_t r = P.ray_begin + rr;
    int v, i, j;
    ray_pixel(r, P.H, P.W, v, i, j);
    const Ray ray = make_ray(P.intr, P.c2w, v, i, j, P.lo, P.hi);
    float t = 0.0f, p[3] = {0.0f, 0.0f, 0.0f};
    int idx[6] = {0, 0, 0, 0, 0, 0};
    float fr[6] = {0, 0, 0, 0, 0, 0};
    if (ray.hit) {
      const float delta = sample_delta(ray, P.N);
      const float u = P.jitter ? jitter_u(P.seed, (uint64_t)r * P.N + k) : 0.5f;
      t = sample_t(ray, delta, k, u);
      sample_p(ray, t, p);
#pragma unroll
      for (int pl = 0; pl < 3; ++pl) {
        const int a = plane_axis_a(pl), b = plane_axis_b(pl);
        if (P.smode == 0) {
          texel_coord(p[a], P.lo[a], P.hi[a], P.inv_ext[a], P.R, idx[2 * pl], fr[2 * pl]);
          texel_coord(p[b], P.lo[b], P.hi[b], P.inv_ext[b], P.R, idx[2 * pl + 1], fr[2 * pl + 1]);
        } else {
          texel_coord_hp(p[a], P.lo[a], P.hi[a], P.inv_ext[a], P.R, idx[2 * pl], fr[2 * pl]);
          texel_coord_hp(p[b], P.lo[b], P.hi[b], P.inv_ext[b], P.R, idx[2 * pl + 1], fr[2 * pl + 1]);
        }
      }
    }
    if (t_k) t_k[q] = t;
    if (points) {
      points[3 * q] = p[0];
      points[3 * q + 1] = p[1];
      points[3 * q + 2] = p[2];
    }
#pragma unroll
    for (int e = 0; e < 6; ++e) {
      if (texel) texel[6 * q + e] = idx[e];
      if (frac) frac[6 * q + e] = fr[e];
    }
  }
}

// row f2: Plucker ray map [V][6][H][W] for rays [ray_begin, ray_end).
// One thread per 4 consecutive rays of a view (HBM-bound: 24 B written per ray, nothing
// read but the cameras): origin and unit direction with make_ray's exact IEEE operation
// order (bit-identical), no AABB slab test (the map does not need it), and six planar
// float4 stores per thread -- a warp writes 512 contiguous bytes per component plane.
__device__ __forceinline__ void pixel_ray(const float *__restrict__ intr, const float *__restrict__ c2w,
                                          int v, int i, int j, float o[3], float d[3]) {
  const float *K = intr + 4 * v;
  const float *M = c2w + 12 * v;
  const float xc = __fdiv_rn(__fsub_rn(__fadd_rn(__int2float_rn(j), 0.5f), __ldg(K + 2)), __ldg(K + 0));
  const float yc = __fdiv_rn(__fsub_rn(__fadd_rn(__int2float_rn(i), 0.5f), __ldg(K + 3)), __ldg(K + 1));
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
    d[a] = __fdiv_rn(dw[a], n);
    o[a] = __ldg(M + 4 * a + 3);
  }
}

__device__ __forceinline__ void plucker6(const float o[3], const float d[3], float m[6]) {
  Ray r;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    r.o[a] = o[a];
    r.d[a] = d[a];
  }
#pragma unroll
  for (int c = 0; c < 6; ++c) m[c] = plucker_component(r, c);
}

template <int RPT> struct VecT;
template <> struct VecT<1> { using T = float; };
template <> struct VecT<2> { using T = float2; };
template <> struct VecT<4> { using T = float4; };
__device__ __forceinline__ float vec_of(const float (&m)[1][6], int c) { return m[0][c]; }
__device__ __forceinline__ float2 vec_of(const float (&m)[2][6], int c) { return make_float2(m[0][c], m[1][c]); }
__device__ __forceinline__ float4 vec_of(const float (&m)[4][6], int c) {
  return make_float4(m[0][c], m[1][c], m[2][c], m[3][c]);
}

// vector path: RPT consecutive rays per thread, HW % RPT == 0 and ray_begin, ray_end
// multiples of RPT (every group lies in one view; its outputs are one aligned RPT-wide
// store per plane).  RPT is chosen per launch: wide stores when there are enough rays to
// fill the machine, one ray per thread (more rays in flight) otherwise.
template <int RPT>
__global__ void __launch_bounds__(256) plucker_vec_kernel(const __grid_constant__ RenderParams P, float *out) {
  using V = typename VecT<RPT>::T;
  const int64_t HW = (int64_t)P.H * P.W;
  const int64_t nv = (P.ray_end - P.ray_begin) / RPT;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nv;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r0 = P.ray_begin + RPT * q;
    int v, pix0;
    if (P.ray_end < (int64_t(1) << 31)) {  // 32-bit index math (every realistic launch)
      v = (int)r0 / (int)HW;
      pix0 = (int)r0 - v * (int)HW;
    } else {
      v = (int)(r0 / HW);
      pix0 = (int)(r0 - (int64_t)v * HW);
    }
    float m[RPT][6];
#pragma unroll
    for (int e = 0; e < RPT; ++e) {
      const int pix = pix0 + e;
      const int i = pix / P.W, j = pix - i * P.W;
      float o[3], d[3];
      pixel_ray(P.intr, P.c2w, v, i, j, o, d);
      plucker6(o, d, m[e]);
    }
    V *dst = reinterpret_cast<V *>(out + (int64_t)v * 6 * HW + pix0);
#pragma unroll
    for (int c = 0; c < 6; ++c) __stcs(dst + c * (HW / RPT), vec_of(m, c));
  }
}

cudaError_t launch_plucker(const RenderParams &P, float *out, cudaStream_t st) {
  const int64_t n = P.ray_end - P.ray_begin;
  if (n <= 0) return cudaSuccess;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t HW = (int64_t)P.H * P.W;
  auto fits = [&](int r) {
    return HW % r == 0 && P.ray_begin % r == 0 && P.ray_end % r == 0 &&
           (reinterpret_cast<uintptr_t>(out) & (4u * r - 1)) == 0;
  };
  // rays per thread: float4 stores once every thread of two full waves (2048 threads
  // per SM) has 4 rays; float2 down to half a wave (measured at 8 x 256^2: 6.5 us kernel
  // vs 6.7 / 6.8 for 1 / 4 rays per thread); scalar below
  const int64_t wave = (int64_t)sms * 2048;
  int rpt = (fits(4) && n / 4 >= 2 * wave) ? 4 : (fits(2) && n / 2 >= wave / 2) ? 2 : 1;
  if (const char *f = getenv("DMV3D_PLUCKER_RPT")) {  // A/B override (tools)
    const int r = atoi(f);
    if ((r == 1 || r == 2 || r == 4) && fits(r)) rpt = r;
  }
  const int64_t items = n / rpt;
  int64_t grid = (items + 255) / 256;  // one item per thread (grid-stride only if huge)
  if (grid > (int64_t)sms * 256) grid = (int64_t)sms * 256;
  timer_begin(P.timer, st);
  if (rpt == 4)
    plucker_vec_kernel<4><<<(int)grid, 256, 0, st>>>(P, out);
  else if (rpt == 2)
    plucker_vec_kernel<2><<<(int)grid, 256, 0, st>>>(P, out);
  else
    plucker_vec_kernel<1><<<(int)grid, 256, 0, st>>>(P, out);
  timer_end(P.timer, st);
  return cudaGetLastError();
}

// Interleaved-tile merge.  Packed layout: rank r's k-th tile (tile id
// r + k world over the whole camera set) is block r nmax + k of rgb [.][3][T][T], alpha
// [.][T][T], x_prev [.][3][T][T] (pack writes one rank's blocks 0..nmax-1 of its own
// buffer, unpack reads all ranks' blocks).  One thread per packed pixel.
__global__ void __launch_bounds__(256) tiles_copy_kernel(int V, int H, int W, int T, int rank, int world,
                                                         int64_t nmax, int ddim_views, int pack,
                                                         const float *__restrict__ s_rgb,
                                                         const float *__restrict__ s_alpha,
                                                         const float *__restrict__ s_xp, float *d_rgb,
                                                         float *d_alpha, float *d_xp) {
  const int64_t TT = (int64_t)T * T, HW = (int64_t)H * W;
  const int64_t TH = (H + T - 1) / T, TW = (W + T - 1) / T, ntiles = (int64_t)V * TH * TW;
  const int64_t nranks = pack ? 1 : world;
  const int64_t total = nranks * nmax * TT;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t blk = e / TT, pp = e - blk * TT;
    const int64_t r = pack ? rank : blk / nmax, k = pack ? blk : blk - r * nmax;
    const int64_t tau = r + k * world;
    if (tau >= ntiles) continue;
    const int v = (int)(tau / (TH * TW));
    const int64_t trem = tau - (int64_t)v * TH * TW;
    const int i = (int)(trem / TW) * T + (int)(pp / T), j = (int)(trem % TW) * T + (int)(pp % T);
    if (i >= H || j >= W) continue;
    const int64_t pix = (int64_t)i * W + j;
    const int64_t ia = (int64_t)v * HW + pix, pa = blk * TT + pp;
    if (s_alpha) {
      if (pack) d_alpha[pa] = __ldg(s_alpha + ia);
      else d_alpha[ia] = __ldg(s_alpha + pa);
    }
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      const int64_t img = ((int64_t)v * 3 + ch) * HW + pix, pk = (blk * 3 + ch) * TT + pp;
      if (s_rgb) {
        if (pack) d_rgb[pk] = __ldg(s_rgb + img);
        else d_rgb[img] = __ldg(s_rgb + pk);
      }
      if (s_xp && v < ddim_views) {
        if (pack) d_xp[pk] = __ldg(s_xp + img);
        else d_xp[img] = __ldg(s_xp + pk);
      }
    }
  }
}

cudaError_t launch_tiles_copy(int V, int H, int W, int T, int rank, int world, int ddim_views, bool pack,
                              const float *src_rgb, const float *src_alpha, const float *src_xp,
                              float *dst_rgb, float *dst_alpha, float *dst_xp, cudaStream_t st) {
  const int64_t TH = (H + T - 1) / T, TW = (W + T - 1) / T, ntiles = (int64_t)V * TH * TW;
  const int64_t nmax = (ntiles + world - 1) / world;
  const int64_t total = (pack ? 1 : (int64_t)world) * nmax * T * T;
  if (total <= 0) return cudaSuccess;
  int64_t grid = (total + 255) / 256;
  if (grid > 148 * 16) grid = 148 * 16;
  tiles_copy_kernel<<<(int)grid, 256, 0, st>>>(V, H, W, T, rank, world, nmax, ddim_views, pack ? 1 : 0,
                                               src_rgb, src_alpha, src_xp, dst_rgb, dst_alpha, dst_xp);
  return cudaGetLastError();
}

cudaError_t launch_ray_geometry(const RenderParams &P, float *o_d, float *tn_tf, uint8_t *hit,
                                cudaStream_t st) {
  const int64_t n = P.ray_end - P.ray_begin;
  if (n <= 0) return cudaSuccess;
  const int64_t grid = (n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096;
  ray_geometry_kernel<<<(int)grid, 256, 0, st>>>(P, o_d, tn_tf, hit);
  return cudaGetLastError();
}

cudaError_t launch_sample_points(const RenderParams &P, float *t_k, float *points,
                                 int32_t *texel, float *frac, cudaStream_t st) {
  const int64_t n = (P.ray_end - P.ray_begin) * P.N;
  if (n <= 0) return cudaSuccess;
  const int64_t grid = (n + 255) / 256 < 8192 ? (n + 255) / 256 : 8192;
  sample_points_kernel<<<(int)grid, 256, 0, st>>>(P, t_k, points, texel, frac);
  return cudaGetLastError();
}

}  // namespace dmv3d
