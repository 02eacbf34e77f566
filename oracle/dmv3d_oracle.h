/*
 * dmv3d_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU oracle for the DMV3D renderer R(S_t, c)
 * (Eq. `reconrender`) and the DDIM x0 -> x_{t-1} update
 * (PAPER.md:25-34, :45-46, :115).  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant with the CUDA product path
 * (paper_2605_18052_b200/csrc, include/dmv3d.h).
 *
 * Precision contract:
 *   - geometry (ray origin/direction, slab test, t_k, sample points, texel
 *     index and fractions) is fp32 with one IEEE-rounded operation per step,
 *     no FMA contraction (-ffp-contract=off), correctly rounded / and sqrt;
 *   - everything after the texel indices (bilinear blend, aggregation, MLP,
 *     compositing, DDIM) is fp64, inputs upcast exactly.
 *
 * Layouts (all row-major, C order):
 *   intrinsics [V][4]       fx, fy, cx, cy  (pixels)
 *   c2w        [V][3][4]    camera-to-world, OpenCV axes (x right, y down, z fwd)
 *   triplane   [3][R][R][C] planes XY, XZ, YZ; [plane][row][col][channel]
 *   W_l        [out][in],   b_l [out]
 *   rgb        [V][3][H][W], alpha [V][H][W]
 */
#ifndef DMV3D_ORACLE_H
#define DMV3D_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define ORC_AGG_MEAN 0
#define ORC_AGG_SUM 1
#define ORC_AGG_CONCAT 2
#define ORC_SAMPLE_ALIGN_CORNERS 0
#define ORC_SAMPLE_HALFPIXEL_ZEROS 1
#define ORC_ACT_RELU 0
#define ORC_ACT_SILU 1
#define ORC_ACT_SOFTPLUS 2

typedef struct {
  int32_t res, channels;
  const double *data; /* [3][res][res][channels] (bf16/fp32 inputs upcast exactly) */
  float aabb_min[3], aabb_max[3];
  int32_t sample_mode; /* ORC_SAMPLE_* (A3; half-pixel + zero padding is row f4) */
} orc_triplane;

typedef struct {
  int32_t num_layers, in_dim, hidden;
  const double *const *weights; /* L pointers, W_l [out][in] (inputs upcast exactly) */
  const double *const *biases;  /* L pointers, b_l [out]     */
  int32_t hidden_act;
  double density_shift, rgb_widen_eps;
} orc_mlp;

typedef struct {
  int32_t num_views, height, width;
  const float *intrinsics, *c2w;
} orc_cameras;

typedef struct {
  int32_t samples_per_ray, agg, jitter;
  uint64_t seed;
  double bg[3];
} orc_render_opts;

/* iDDPM cosine schedule, 0-based alpha_bar[t], t in [0,T). */
void orc_cosine_alpha_bar(int32_t T, double s, double *alpha_bar);

/* fp32 geometry for one ray id r = (v*H + i)*W + j (C1 steps 1-2). */
void orc_ray_geometry(const orc_cameras *cams, const float aabb_min[3],
                      const float aabb_max[3], int64_t r, float o[3], float d[3],
                      float *t_near, float *t_far, int32_t *hit);

/* Plucker ray (o x d, d) of ray id r, fp32. */
void orc_plucker(const orc_cameras *cams, int64_t r, float out[6]);

/* in-kernel DDIM noise (row f4): standard normal for element e of x_t. */
double orc_noise(uint64_t seed, uint64_t e);

/* portable jitter value u in [0,1) for sample id (ray*N + k) (A10). */
float orc_jitter(uint64_t seed, uint64_t sample_id);

/* fp32 sample parameter t_k and point p_k (C1 step 3). */
void orc_sample_point(const float o[3], const float d[3], float t_near, float t_far,
                      int32_t N, int32_t k, int32_t jitter, uint64_t seed, int64_t r,
                      float *t_k, float p[3]);

/* fp32 texel index/fraction for coordinate q on an axis [lo,hi] (align corners). */
void orc_texel_coord(float q, float lo, float hi, int32_t R, int32_t *i0, float *f);
void orc_texel_coord_halfpixel(float q, float lo, float hi, int32_t R, int32_t *i0, float *f);

/* aggregated triplane feature at point p, fp64 out [K] (C1 step 4). */
void orc_point_features(const orc_triplane *tp, int32_t agg, const float p[3], double *out);

/* shared MLP decode of feature h0[K] -> sigma, rgb[3] (C1 step 5). */
void orc_mlp_decode(const orc_mlp *mlp, const double *h0, double *sigma, double rgb[3]);

/* full decode at a point: gather + MLP. out[4] = sigma, r, g, b */
void orc_decode_point(const orc_triplane *tp, const orc_mlp *mlp, int32_t agg,
                      const float p[3], double out[4]);

/* density grid (row f3): grid point idx -> p (fp32, align-corners over the box) */
void orc_grid_point(const float lo[3], const float hi[3], int32_t G, int64_t idx, float p[3]);
/* sigma [G][G][G] (x fastest), rgb [3][G][G][G] or NULL; fp64 */
void orc_density_grid(const orc_triplane *tp, const orc_mlp *mlp, int32_t agg, int32_t G,
                      double *sigma, double *rgb, int32_t num_threads);

/* renderer backward (row f1): dL/dS and dL/dMLP for L = <g, rgb> + <gA, alpha>,
 * accumulated (fp64) into dF [3][R][R][C], dW[l] [out][in], db[l] [out]. */
void orc_render_ray_backward(const orc_triplane *tp, const orc_cameras *cams,
                             const orc_mlp *mlp, const orc_render_opts *opts, int64_t r,
                             const double g[3], double gA, double *dF, double *const *dW,
                             double *const *db);
void orc_render_backward(const orc_triplane *tp, const orc_cameras *cams, const orc_mlp *mlp,
                         const orc_render_opts *opts, const double *grad_rgb,
                         const double *grad_alpha, double *dF, double *const *dW,
                         double *const *db);

/* render one ray (no early termination): rgb[3], alpha. */
void orc_render_ray(const orc_triplane *tp, const orc_cameras *cams, const orc_mlp *mlp,
                    const orc_render_opts *opts, int64_t r, double rgb[3], double *alpha);

/* render a list of ray ids (OpenMP over rays). rgb [n][3], alpha [n]. */
void orc_render_rays(const orc_triplane *tp, const orc_cameras *cams, const orc_mlp *mlp,
                     const orc_render_opts *opts, int64_t n, const int64_t *ray_ids,
                     double *rgb, double *alpha, int32_t num_threads);

/* render all views: rgb [V][3][H][W], alpha [V][H][W] (fp64). */
void orc_render_views(const orc_triplane *tp, const orc_cameras *cams, const orc_mlp *mlp,
                      const orc_render_opts *opts, double *rgb, double *alpha,
                      int32_t num_threads);

/* DDIM x0 -> x_{t-1} (A15-A20), elementwise over
 * [V][3][H][W]; x0_rgb is the rendered image; z may be NULL iff eta == 0;
 * keep_mask [V] or NULL. */
void orc_ddim_step(const double *alpha_bar, int32_t T, int32_t t, int32_t t_prev, double eta,
                   double x0_scale, double x0_shift, int32_t V, int32_t H, int32_t W,
                   const double *x_t, const double *x0_rgb, const double *z,
                   const uint8_t *keep_mask, double *x_prev);

#ifdef __cplusplus
}
#endif
#endif
