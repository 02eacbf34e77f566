/*
 * dmv3d_oracle.c -- TEST INFRASTRUCTURE ONLY (see dmv3d_oracle.h).
 *
 * A plain CPU transcription of what the DMV3D renderer and DDIM step compute,
 * written from PAPER.md and the readings in DESIGN.md ("Readings of the
 * paper").  No blocking, fusion, early termination or
 * reordering: every ray marches every sample, every sample evaluates the
 * full MLP, the transmittance is a plain sequential product.
 *
 * Build: gcc -O2 -fopenmp -ffp-contract=off -fPIC -shared (no -ffast-math).
 * Parity pins live in tests/test_oracle_*.py (closed forms, brute force,
 * library special cases); see DESIGN.md "Oracle pins".
 */
#include "dmv3d_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------ */
/* Schedule: "add noise according to a cosine schedule", */
/* T = 1000 ("t=980/1000").  Reading A16: iDDPM cosine,  */
/* f(t) = cos^2(((t/T)+s)/(1+s) * pi/2), beta_j = min(1 - f(j+1)/f(j), */
/* 0.999), alpha_bar_t = prod_{j<=t} (1 - beta_j), 0-based t.          */
/* ------------------------------------------------------------------ */
static double cosine_f(double t, double T, double s) {
  double a = ((t / T) + s) / (1.0 + s) * (M_PI / 2.0);
  double c = cos(a);
  return c * c;
}

void orc_cosine_alpha_bar(int32_t T, double s, double *alpha_bar) {
  double prod = 1.0;
  for (int32_t j = 0; j < T; ++j) {
    double beta = 1.0 - cosine_f(j + 1, T, s) / cosine_f(j, T, s);
    if (beta > 0.999) beta = 0.999;
    prod = prod * (1.0 - beta);
    alpha_bar[j] = prod;
  }
}

/* ------------------------------------------------------------------ */
/* Ray generation (reading A8): pinhole, pixel centres at +1/2, OpenCV  */
/* camera axes, unit direction; origin = camera centre.  Plucker rays  */
/* "o and d ... computed from the camera parameters".    */
/* Slab test on the object box [-1,1]^3 (A9).      */
/* fp32, one rounding per line (C1 steps 1-2).                          */
/* ------------------------------------------------------------------ */
void orc_ray_geometry(const orc_cameras *cams, const float aabb_min[3],
                      const float aabb_max[3], int64_t r, float o[3], float d[3],
                      float *t_near, float *t_far, int32_t *hit) {
  const int64_t HW = (int64_t)cams->height * cams->width;
  const int64_t v = r / HW;
  const int64_t rem = r - v * HW;
  const int64_t i = rem / cams->width;
  const int64_t j = rem - i * cams->width;
  const float *K = cams->intrinsics + 4 * v;
  const float *M = cams->c2w + 12 * v;

  float px = (float)j + 0.5f;
  float py = (float)i + 0.5f;
  float xc = (px - K[2]) / K[0];
  float yc = (py - K[3]) / K[1];

  float dw[3];
  for (int a = 0; a < 3; ++a) {
    float m0 = M[4 * a + 0] * xc;
    float m1 = M[4 * a + 1] * yc;
    float s = m0 + m1;
    dw[a] = s + M[4 * a + 2];
  }
  float q0 = dw[0] * dw[0];
  float q1 = dw[1] * dw[1];
  float q2 = dw[2] * dw[2];
  float nn = (q0 + q1) + q2;
  float n = sqrtf(nn);
  for (int a = 0; a < 3; ++a) {
    d[a] = dw[a] / n;
    o[a] = M[4 * a + 3];
  }

  int32_t ok = 1;
  float tmin[3], tmax[3];
  for (int a = 0; a < 3; ++a) {
    float lo = aabb_min[a], hi = aabb_max[a];
    if (d[a] == 0.0f) {
      if (o[a] < lo || o[a] > hi) ok = 0;
      tmin[a] = -INFINITY;
      tmax[a] = INFINITY;
    } else {
      float t0 = (lo - o[a]) / d[a];
      float t1 = (hi - o[a]) / d[a];
      tmin[a] = fminf(t0, t1);
      tmax[a] = fmaxf(t0, t1);
    }
  }
  float tn = fmaxf(fmaxf(fmaxf(tmin[0], tmin[1]), tmin[2]), 0.0f);
  float tf = fminf(fminf(tmax[0], tmax[1]), tmax[2]);
  if (ok && tf > tn) {
    *t_near = tn;
    *t_far = tf;
    *hit = 1;
  } else {
    *t_near = 0.0f;
    *t_far = 0.0f;
    *hit = 0;
  }
}

/* Plucker coordinates of a pixel ray, r = (o x d, d) (LFN),  */
/* fp32, each component two rounded products and one rounded difference. */
void orc_plucker(const orc_cameras *cams, int64_t r, float out[6]) {
  const float lo[3] = {-1.0f, -1.0f, -1.0f}, hi[3] = {1.0f, 1.0f, 1.0f};
  float o[3], d[3], tn, tf;
  int32_t hit;
  orc_ray_geometry(cams, lo, hi, r, o, d, &tn, &tf, &hit);
  float a, b;
  a = o[1] * d[2];
  b = o[2] * d[1];
  out[0] = a - b;
  a = o[2] * d[0];
  b = o[0] * d[2];
  out[1] = a - b;
  a = o[0] * d[1];
  b = o[1] * d[0];
  out[2] = a - b;
  out[3] = d[0];
  out[4] = d[1];
  out[5] = d[2];
}

/* Reading A10: optional stratified jitter from a portable counter-based */
/* generator (splitmix64 finaliser).                    */
float orc_jitter(uint64_t seed, uint64_t sample_id) {
  uint64_t z = seed + (sample_id + 1ull) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z = z ^ (z >> 31);
  return (float)(z >> 40) * (1.0f / 16777216.0f);
}

/* Row f4: in-kernel DDIM noise z (fresh noise per step,     */
/* :1102) from the same splitmix64 counter hash: element e of x_t draws   */
/* u1 = (h(seed, 2e) >> 40 + 1) 2^-24 in (0,1], u2 = (h(seed, 2e+1) >> 40) */
/* 2^-24 in [0,1) and z = sqrt(-2 ln u1) cos(2 pi u2) (Box-Muller), fp64.  */
double orc_noise(uint64_t seed, uint64_t e) {
  uint64_t z1 = seed + (2 * e + 1ull) * 0x9E3779B97F4A7C15ull;
  z1 = (z1 ^ (z1 >> 30)) * 0xBF58476D1CE4E5B9ull;
  z1 = (z1 ^ (z1 >> 27)) * 0x94D049BB133111EBull;
  z1 = z1 ^ (z1 >> 31);
  uint64_t z2 = seed + (2 * e + 2ull) * 0x9E3779B97F4A7C15ull;
  z2 = (z2 ^ (z2 >> 30)) * 0xBF58476D1CE4E5B9ull;
  z2 = (z2 ^ (z2 >> 27)) * 0x94D049BB133111EBull;
  z2 = z2 ^ (z2 >> 31);
  const double u1 = (double)((z1 >> 40) + 1) / 16777216.0;
  const double u2 = (double)(z2 >> 40) / 16777216.0;
  return sqrt(-2.0 * log(u1)) * cos(2.0 * M_PI * u2);
}

/* Samples: N intervals partition [t_near, t_far] (A10, A11).          */
void orc_sample_point(const float o[3], const float d[3], float t_near, float t_far,
                      int32_t N, int32_t k, int32_t jitter, uint64_t seed, int64_t r,
                      float *t_k, float p[3]) {
  float delta = (t_far - t_near) / (float)N;
  float u = jitter ? orc_jitter(seed, (uint64_t)r * (uint64_t)N + (uint64_t)k) : 0.5f;
  float kk = (float)k + u;
  float step = kk * delta;
  float t = t_near + step;
  *t_k = t;
  for (int a = 0; a < 3; ++a) {
    float m = t * d[a];
    p[a] = o[a] + m;
  }
}

/* Reading A3: align-corners texel addressing, clamp to the plane.      */
void orc_texel_coord(float q, float lo, float hi, int32_t R, int32_t *i0, float *f) {
  float ext = hi - lo;
  float s = (q - lo) / ext;
  float px = s * (float)(R - 1);
  px = fminf(fmaxf(px, 0.0f), (float)(R - 1));
  int32_t ix = (int32_t)floorf(px);
  if (ix > R - 2) ix = R - 2;
  *i0 = ix;
  *f = px - (float)ix;
}

/* Row f4 variant: half-pixel texel centres with zero padding (the        */
/* convention of grid_sample(align_corners=False, padding_mode='zeros')):  */
/* px = ((q - lo)/(hi - lo)) R - 1/2, i0 = floor(px) in [-1, R-1], no      */
/* clamp; texels outside the plane read as 0.                              */
void orc_texel_coord_halfpixel(float q, float lo, float hi, int32_t R, int32_t *i0, float *f) {
  float ext = hi - lo;
  float s = (q - lo) / ext;
  float a = s * (float)R;
  float px = a - 0.5f;
  int32_t ix = (int32_t)floorf(px);
  *i0 = ix;
  *f = px - (float)ix;
}

static void texel_coord_mode(const orc_triplane *tp, int axis, float q, int32_t *i0, float *f) {
  if (tp->sample_mode == ORC_SAMPLE_HALFPIXEL_ZEROS)
    orc_texel_coord_halfpixel(q, tp->aabb_min[axis], tp->aabb_max[axis], tp->res, i0, f);
  else
    orc_texel_coord(q, tp->aabb_min[axis], tp->aabb_max[axis], tp->res, i0, f);
}

/* texel (row, col) of plane pl, or NULL outside the plane (zero padding) */
static const double *texel(const orc_triplane *tp, int pl, int32_t row, int32_t col) {
  const int32_t R = tp->res;
  if (row < 0 || row >= R || col < 0 || col >= R) return NULL;
  return tp->data + (((size_t)pl * R + row) * R + col) * tp->channels;
}

/* ------------------------------------------------------------------ */
/* Triplane NeRF features (A2-A4): planes XY,   */
/* XZ, YZ; plane (a,b): column <- axis a, row <- axis b; bilinear       */
/* interpolation of the 4 texels; mean (or sum) over the 3 planes, or   */
/* their concatenation (row f4).                                        */
/* ------------------------------------------------------------------ */
static const int PLANE_AXES[3][2] = {{0, 1}, {0, 2}, {1, 2}};

void orc_point_features(const orc_triplane *tp, int32_t agg, const float p[3], double *out) {
  const int32_t C = tp->channels;
  const int32_t K = agg == ORC_AGG_CONCAT ? 3 * C : C;
  for (int32_t c = 0; c < K; ++c) out[c] = 0.0;
  for (int pl = 0; pl < 3; ++pl) {
    int a = PLANE_AXES[pl][0], b = PLANE_AXES[pl][1];
    int32_t ix, iy;
    float fxf, fyf;
    texel_coord_mode(tp, a, p[a], &ix, &fxf);
    texel_coord_mode(tp, b, p[b], &iy, &fyf);
    double fx = (double)fxf, fy = (double)fyf;
    const double w[4] = {(1.0 - fx) * (1.0 - fy), fx * (1.0 - fy), (1.0 - fx) * fy, fx * fy};
    const double *t[4] = {texel(tp, pl, iy, ix), texel(tp, pl, iy, ix + 1),
                          texel(tp, pl, iy + 1, ix), texel(tp, pl, iy + 1, ix + 1)};
    double *dst = out + (agg == ORC_AGG_CONCAT ? pl * C : 0);
    for (int32_t c = 0; c < C; ++c) {
      double v = 0.0;
      for (int e = 0; e < 4; ++e)
        if (t[e]) v += w[e] * t[e][c];
      dst[c] += v;
    }
  }
  if (agg == ORC_AGG_MEAN)
    for (int32_t c = 0; c < C; ++c) out[c] = out[c] / 3.0;
}

/* ------------------------------------------------------------------ */
/* Shared MLP to density and colour (A5-A7).         */
/* ------------------------------------------------------------------ */
static double softplus(double x) { return log1p(exp(-fabs(x))) + (x > 0.0 ? x : 0.0); }
static double sigmoid(double x) { return 1.0 / (1.0 + exp(-x)); }
static double hidden_act(int32_t kind, double x) {
  switch (kind) {
    case ORC_ACT_SILU: return x * sigmoid(x);
    case ORC_ACT_SOFTPLUS: return softplus(x);
    default: return x > 0.0 ? x : 0.0;
  }
}

void orc_mlp_decode(const orc_mlp *mlp, const double *h0, double *sigma, double rgb[3]) {
  const int32_t L = mlp->num_layers;
  int32_t maxw = mlp->in_dim > mlp->hidden ? mlp->in_dim : mlp->hidden;
  if (maxw < 4) maxw = 4;
  double *cur = (double *)malloc(sizeof(double) * maxw);
  double *nxt = (double *)malloc(sizeof(double) * maxw);
  memcpy(cur, h0, sizeof(double) * mlp->in_dim);
  int32_t in = mlp->in_dim;
  for (int32_t l = 0; l < L; ++l) {
    int32_t out = (l == L - 1) ? 4 : mlp->hidden;
    const double *Wl = mlp->weights[l];
    const double *bl = mlp->biases[l];
    for (int32_t o = 0; o < out; ++o) {
      double acc = bl[o];
      for (int32_t q = 0; q < in; ++q) acc += Wl[(size_t)o * in + q] * cur[q];
      nxt[o] = (l == L - 1) ? acc : hidden_act(mlp->hidden_act, acc);
    }
    double *tmp = cur;
    cur = nxt;
    nxt = tmp;
    in = out;
  }
  *sigma = softplus(cur[0] + mlp->density_shift);
  for (int c = 0; c < 3; ++c) {
    double s = sigmoid(cur[1 + c]);
    rgb[c] = s * (1.0 + 2.0 * mlp->rgb_widen_eps) - mlp->rgb_widen_eps;
  }
  free(cur);
  free(nxt);
}

void orc_decode_point(const orc_triplane *tp, const orc_mlp *mlp, int32_t agg,
                      const float p[3], double out[4]) {
  double *h0 = (double *)malloc(sizeof(double) * 3 * tp->channels); /* concat: 3C */
  orc_point_features(tp, agg, p, h0);
  double sigma, rgb[3];
  orc_mlp_decode(mlp, h0, &sigma, rgb);
  out[0] = sigma;
  out[1] = rgb[0];
  out[2] = rgb[1];
  out[3] = rgb[2];
  free(h0);
}

/* Density grid for marching cubes ("CD ... marching cubes on   */
/* the NeRF density"): G^3 points on the box, align-corners,    */
/* p_a = lo_a + (idx_a / (G-1)) (hi_a - lo_a) in fp32; x fastest.              */
void orc_grid_point(const float lo[3], const float hi[3], int32_t G, int64_t idx, float p[3]) {
  const int64_t ix = idx % G, iy = (idx / G) % G, iz = idx / ((int64_t)G * G);
  const int64_t id3[3] = {ix, iy, iz};
  for (int a = 0; a < 3; ++a) {
    float s = (float)id3[a] / (float)(G - 1);
    float ext = hi[a] - lo[a];
    float m = s * ext;
    p[a] = lo[a] + m;
  }
}

void orc_density_grid(const orc_triplane *tp, const orc_mlp *mlp, int32_t agg, int32_t G,
                      double *sigma, double *rgb, int32_t num_threads) {
  const int64_t n = (int64_t)G * G * G;
#ifdef _OPENMP
  if (num_threads > 0) omp_set_num_threads(num_threads);
#pragma omp parallel for schedule(dynamic, 64)
#endif
  for (int64_t q = 0; q < n; ++q) {
    float p[3];
    orc_grid_point(tp->aabb_min, tp->aabb_max, G, q, p);
    double out[4];
    orc_decode_point(tp, mlp, agg, p, out);
    sigma[q] = out[0];
    if (rgb)
      for (int c = 0; c < 3; ++c) rgb[c * n + q] = out[1 + c];
  }
}

/* ------------------------------------------------------------------ */
/* Volume rendering quadrature (A11-A13):             */
/* tau_k = sigma_k * delta, alpha_k = 1 - exp(-tau_k), T_0 = 1,         */
/* T_{k+1} = T_k exp(-tau_k), w_k = T_k alpha_k,                        */
/* rgb = sum_k w_k c_k + T_N bg, A = 1 - T_N.  No early termination.    */
/* ------------------------------------------------------------------ */
void orc_render_ray(const orc_triplane *tp, const orc_cameras *cams, const orc_mlp *mlp,
                    const orc_render_opts *opts, int64_t r, double rgb[3], double *alpha) {
  float o[3], d[3], tn, tf;
  int32_t hit;
  orc_ray_geometry(cams, tp->aabb_min, tp->aabb_max, r, o, d, &tn, &tf, &hit);
  if (!hit) {
    rgb[0] = opts->bg[0];
    rgb[1] = opts->bg[1];
    rgb[2] = opts->bg[2];
    *alpha = 0.0;
    return;
  }
  const int32_t N = opts->samples_per_ray;
  const double delta = (double)((tf - tn) / (float)N);
  double T = 1.0, acc[3] = {0.0, 0.0, 0.0};
  double *h0 = (double *)malloc(sizeof(double) * 3 * tp->channels); /* concat: 3C */
  for (int32_t k = 0; k < N; ++k) {
    float tk, p[3];
    orc_sample_point(o, d, tn, tf, N, k, opts->jitter, opts->seed, r, &tk, p);
    orc_point_features(tp, opts->agg, p, h0);
    double sigma, c[3];
    orc_mlp_decode(mlp, h0, &sigma, c);
    double tau = sigma * delta;
    double a = -expm1(-tau);
    double w = T * a;
    for (int ch = 0; ch < 3; ++ch) acc[ch] += w * c[ch];
    T = T * exp(-tau);
  }
  free(h0);
  for (int ch = 0; ch < 3; ++ch) rgb[ch] = acc[ch] + T * opts->bg[ch];
  *alpha = 1.0 - T;
}

/* ------------------------------------------------------------------ */
/* Renderer backward: "differentiable volume rendering"  */
/* supervised by L_recon.  For one ray,  */
/* the gradient of L = sum_ch g_ch rgb_ch + gA alpha w.r.t. the triplane */
/* and the MLP parameters, by the chain rule through the quadrature:     */
/*   dC/dtau_k = T_{k+1} c_k - R_k, R_k = sum_{j>k} w_j c_j + T_N bg,    */
/*   dA/dtau_k = T_N, dC/dc_k = w_k, tau_k = sigma_k delta;              */
/* sample positions (hence delta and the texel cells) are constants.     */
/* Accumulates into dF [3][R][R][C], dW[l] [out][in], db[l] [out].       */
/* ------------------------------------------------------------------ */
static double hidden_act_grad(int32_t kind, double z) {
  switch (kind) {
    case ORC_ACT_SILU: {
      double s = sigmoid(z);
      return s + z * s * (1.0 - s);
    }
    case ORC_ACT_SOFTPLUS: return sigmoid(z);
    default: return z > 0.0 ? 1.0 : 0.0;
  }
}

void orc_render_ray_backward(const orc_triplane *tp, const orc_cameras *cams,
                             const orc_mlp *mlp, const orc_render_opts *opts, int64_t r,
                             const double g[3], double gA, double *dF, double *const *dW,
                             double *const *db) {
  float o[3], d[3], tn, tf;
  int32_t hit;
  orc_ray_geometry(cams, tp->aabb_min, tp->aabb_max, r, o, d, &tn, &tf, &hit);
  if (!hit) return;
  const int32_t N = opts->samples_per_ray, L = mlp->num_layers, K = mlp->in_dim,
                H = mlp->hidden, R = tp->res, C = tp->channels;
  const double delta = (double)((tf - tn) / (float)N);
  /* per-sample storage: layer inputs h_0..h_{L-1} (h_0: K wide, others H), the
     pre-activations z_1..z_{L-1} (H), the 4 outputs */
  const int32_t S = K + (L - 1) * H + (L - 1) * H + 4;
  double *buf = (double *)calloc((size_t)N * S, sizeof(double));
  double *sig = (double *)malloc(sizeof(double) * N), *col = (double *)malloc(sizeof(double) * 3 * N);
  float *pts = (float *)malloc(sizeof(float) * 3 * N);
#define H_IN(k, l) (buf + (size_t)(k) * S + ((l) == 0 ? 0 : K + ((l) - 1) * H))
#define Z_OF(k, l) (buf + (size_t)(k) * S + K + (L - 1) * H + ((l) - 1) * H) /* z_l, l>=1 */
#define OUT(k) (buf + (size_t)(k) * S + K + 2 * (L - 1) * H)
  for (int32_t k = 0; k < N; ++k) {
    float tk;
    orc_sample_point(o, d, tn, tf, N, k, opts->jitter, opts->seed, r, &tk, pts + 3 * k);
    orc_point_features(tp, opts->agg, pts + 3 * k, H_IN(k, 0));
    for (int32_t l = 0; l < L; ++l) {
      const int32_t in = l == 0 ? K : H, out = l == L - 1 ? 4 : H;
      const double *h = H_IN(k, l);
      for (int32_t q = 0; q < out; ++q) {
        double acc = mlp->biases[l][q];
        for (int32_t i = 0; i < in; ++i) acc += mlp->weights[l][(size_t)q * in + i] * h[i];
        if (l == L - 1) {
          OUT(k)[q] = acc;
        } else {
          Z_OF(k, l + 1)[q] = acc;
          H_IN(k, l + 1)[q] = hidden_act(mlp->hidden_act, acc);
        }
      }
    }
    sig[k] = softplus(OUT(k)[0] + mlp->density_shift);
    for (int c = 0; c < 3; ++c)
      col[3 * k + c] =
          sigmoid(OUT(k)[1 + c]) * (1.0 + 2.0 * mlp->rgb_widen_eps) - mlp->rgb_widen_eps;
  }
  /* forward quadrature */
  double *T = (double *)malloc(sizeof(double) * (N + 1)), *w = (double *)malloc(sizeof(double) * N);
  T[0] = 1.0;
  for (int32_t k = 0; k < N; ++k) {
    const double tau = sig[k] * delta;
    w[k] = T[k] * (-expm1(-tau));
    T[k + 1] = T[k] * exp(-tau);
  }
  /* R_k suffix sums, then backward per sample */
  double Rk[3];
  for (int c = 0; c < 3; ++c) Rk[c] = T[N] * opts->bg[c];
  double *dh = (double *)malloc(sizeof(double) * (K > H ? K : H));
  double *delta_v = (double *)malloc(sizeof(double) * (H > 4 ? H : 4));
  for (int32_t k = N - 1; k >= 0; --k) {
    double dtau = gA * T[N];
    for (int c = 0; c < 3; ++c) dtau += g[c] * (T[k + 1] * col[3 * k + c] - Rk[c]);
    for (int c = 0; c < 3; ++c) Rk[c] += w[k] * col[3 * k + c];
    const double s0 = sigmoid(OUT(k)[0] + mlp->density_shift);
    delta_v[0] = dtau * delta * s0;
    for (int c = 0; c < 3; ++c) {
      const double s = sigmoid(OUT(k)[1 + c]);
      delta_v[1 + c] = g[c] * w[k] * (1.0 + 2.0 * mlp->rgb_widen_eps) * s * (1.0 - s);
    }
    for (int32_t l = L - 1; l >= 0; --l) {
      const int32_t in = l == 0 ? K : H, out = l == L - 1 ? 4 : H;
      const double *h = H_IN(k, l);
      for (int32_t q = 0; q < out; ++q) {
        db[l][q] += delta_v[q];
        for (int32_t i = 0; i < in; ++i) dW[l][(size_t)q * in + i] += delta_v[q] * h[i];
      }
      for (int32_t i = 0; i < in; ++i) {
        double acc = 0.0;
        for (int32_t q = 0; q < out; ++q) acc += mlp->weights[l][(size_t)q * in + i] * delta_v[q];
        dh[i] = acc;
      }
      if (l > 0)
        for (int32_t i = 0; i < in; ++i) delta_v[i] = dh[i] * hidden_act_grad(mlp->hidden_act, Z_OF(k, l)[i]);
    }
    /* dh = dL/dh0 -> bilinear corners of the 3 planes */
    const double scale = opts->agg == ORC_AGG_MEAN ? 1.0 / 3.0 : 1.0;
    for (int pl = 0; pl < 3; ++pl) {
      const int a = PLANE_AXES[pl][0], b = PLANE_AXES[pl][1];
      int32_t ix, iy;
      float fxf, fyf;
      texel_coord_mode(tp, a, pts[3 * k + a], &ix, &fxf);
      texel_coord_mode(tp, b, pts[3 * k + b], &iy, &fyf);
      const double fx = fxf, fy = fyf;
      const double wc[4] = {(1 - fx) * (1 - fy), fx * (1 - fy), (1 - fx) * fy, fx * fy};
      const int32_t rr[4] = {iy, iy, iy + 1, iy + 1}, cc4[4] = {ix, ix + 1, ix, ix + 1};
      const double *g = dh + (opts->agg == ORC_AGG_CONCAT ? pl * C : 0);
      for (int e = 0; e < 4; ++e) {
        if (rr[e] < 0 || rr[e] >= R || cc4[e] < 0 || cc4[e] >= R) continue;  /* zero padding */
        const size_t off = ((size_t)(pl * R + rr[e]) * R + cc4[e]) * C;
        for (int32_t c = 0; c < C; ++c) dF[off + c] += scale * wc[e] * g[c];
      }
    }
  }
#undef H_IN
#undef Z_OF
#undef OUT
  free(buf);
  free(sig);
  free(col);
  free(pts);
  free(T);
  free(w);
  free(dh);
  free(delta_v);
}

/* all views: grad_rgb [V][3][H][W], grad_alpha [V][H][W] or NULL; sequential
   (the accumulators are shared by all rays) */
void orc_render_backward(const orc_triplane *tp, const orc_cameras *cams, const orc_mlp *mlp,
                         const orc_render_opts *opts, const double *grad_rgb,
                         const double *grad_alpha, double *dF, double *const *dW,
                         double *const *db) {
  const int64_t HW = (int64_t)cams->height * cams->width;
  const int64_t n = (int64_t)cams->num_views * HW;
  for (int64_t r = 0; r < n; ++r) {
    const int64_t v = r / HW, pix = r - v * HW;
    double g[3];
    for (int c = 0; c < 3; ++c) g[c] = grad_rgb[(v * 3 + c) * HW + pix];
    const double gA = grad_alpha ? grad_alpha[r] : 0.0;
    orc_render_ray_backward(tp, cams, mlp, opts, r, g, gA, dF, dW, db);
  }
}

void orc_render_rays(const orc_triplane *tp, const orc_cameras *cams, const orc_mlp *mlp,
                     const orc_render_opts *opts, int64_t n, const int64_t *ray_ids,
                     double *rgb, double *alpha, int32_t num_threads) {
#ifdef _OPENMP
  if (num_threads > 0) omp_set_num_threads(num_threads);
#pragma omp parallel for schedule(dynamic, 16)
#endif
  for (int64_t q = 0; q < n; ++q) {
    double c[3], a;
    orc_render_ray(tp, cams, mlp, opts, ray_ids[q], c, &a);
    rgb[3 * q + 0] = c[0];
    rgb[3 * q + 1] = c[1];
    rgb[3 * q + 2] = c[2];
    alpha[q] = a;
  }
}

void orc_render_views(const orc_triplane *tp, const orc_cameras *cams, const orc_mlp *mlp,
                      const orc_render_opts *opts, double *rgb, double *alpha,
                      int32_t num_threads) {
  const int64_t HW = (int64_t)cams->height * cams->width;
  const int64_t nrays = (int64_t)cams->num_views * HW;
#ifdef _OPENMP
  if (num_threads > 0) omp_set_num_threads(num_threads);
#pragma omp parallel for schedule(dynamic, 16)
#endif
  for (int64_t r = 0; r < nrays; ++r) {
    double c[3], a;
    orc_render_ray(tp, cams, mlp, opts, r, c, &a);
    int64_t v = r / HW, pix = r - v * HW;
    for (int ch = 0; ch < 3; ++ch) rgb[(v * 3 + ch) * HW + pix] = c[ch];
    if (alpha) alpha[r] = a;
  }
}

/* ------------------------------------------------------------------ */
/* DDIM update from the x0 prediction (A15-A20):  */
/* x0 = scale*rgb + shift; eps = (x_t - sqrt(ab_t) x0)/sqrt(1-ab_t);    */
/* sigma_t = eta sqrt((1-ab_p)/(1-ab_t)) sqrt(1-ab_t/ab_p);             */
/* x_{t-1} = sqrt(ab_p) x0 + sqrt(1-ab_p-sigma_t^2) eps + sigma_t z;    */
/* ab_p = 1 when t_prev < 0; keep_mask views stay noise-free.    */
/* ------------------------------------------------------------------ */
void orc_ddim_step(const double *alpha_bar, int32_t T, int32_t t, int32_t t_prev, double eta,
                   double x0_scale, double x0_shift, int32_t V, int32_t H, int32_t W,
                   const double *x_t, const double *x0_rgb, const double *z,
                   const uint8_t *keep_mask, double *x_prev) {
  (void)T;
  const double ab_t = alpha_bar[t];
  const double ab_p = (t_prev >= 0) ? alpha_bar[t_prev] : 1.0;
  const double sigma_t = eta * sqrt((1.0 - ab_p) / (1.0 - ab_t)) * sqrt(1.0 - ab_t / ab_p);
  double c2 = 1.0 - ab_p - sigma_t * sigma_t;
  if (c2 < 0.0) c2 = 0.0;
  const double c_eps = sqrt(c2);
  const int64_t per_view = (int64_t)3 * H * W;
  for (int32_t v = 0; v < V; ++v) {
    for (int64_t e = 0; e < per_view; ++e) {
      int64_t idx = (int64_t)v * per_view + e;
      if (keep_mask && keep_mask[v]) {
        x_prev[idx] = x_t[idx];
        continue;
      }
      double x0 = x0_scale * x0_rgb[idx] + x0_shift;
      double eps = (x_t[idx] - sqrt(ab_t) * x0) / sqrt(1.0 - ab_t);
      double xp = sqrt(ab_p) * x0 + c_eps * eps;
      if (sigma_t != 0.0) xp += sigma_t * z[idx];
      x_prev[idx] = xp;
    }
  }
}
