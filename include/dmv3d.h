/*
 * dmv3d.h -- C ABI of libdmv3d.so: the B200 (sm_100a) hot path of DMV3D's
 * reconstruction-based multi-view denoiser (arXiv 2605.18052, PAPER.md).
 *
 *   I_{r,t} = R(S_t, c)                                   (Eq. reconrender)
 *   x_t = sqrt(ab_t) x_0 + sqrt(1 - ab_t) eps
 *   x0-prediction -> x_{t-1} (DDIM)
 *
 * R is the triplane-NeRF renderer (Instant3D LRM
 * PAPER.md:544): ray generation from the camera set C (a1), ray/AABB slab
 * test on the object box [-1,1]^3 and N midpoint samples (a2),
 * bilinear gather from the three axis-aligned planes with mean aggregation
 * (a3), the shared MLP decoder to density and colour (a4), front-to-back
 * compositing (a5); the DDIM step (a6) maps the rendered views to x_{t-1}.
 * Every reading of the paper the library relies on is listed in DESIGN.md
 * ("Readings") with its id (A1..A25).
 *
 * Conventions (all entry points)
 * ------------------------------
 *  - Tensor pointers are DEVICE pointers on the current CUDA device unless a
 *    field says HOST.  The caller owns every buffer; the library allocates
 *    no device memory on these calls (the *_host variant below uses a
 *    caller-created workspace).  Inputs must stay valid until the work
 *    enqueued on `stream` completes.
 *  - Calls enqueue on `stream` (a cudaStream_t, 0 = legacy default stream)
 *    and never synchronise the host.  Launch errors are returned at once as
 *    DMV3D_ERR_CUDA; faults inside kernels surface at the caller's next sync.
 *  - On any non-OK status nothing has been enqueued and dmv3d_last_error()
 *    returns a thread-local message.  Re-entrant; no global mutable state.
 *  - Layouts are C-order (row-major):
 *      intrinsics [V][4]  fx, fy, cx, cy in pixels (pinhole, pixel centres at +1/2)
 *      c2w        [V][3][4] camera-to-world, OpenCV axes (x right, y down, z forward)
 *      triplane   [3][R][R][C] channels-last; planes XY, XZ, YZ; plane (a,b):
 *                 column <- axis a, row <- axis b; align-corners texels
 *      W_l        [out][in] (PyTorch nn.Linear), b_l [out] fp32
 *      images     rgb [V][3][H][W], alpha [V][H][W], x_t / z / x_prev
 *                 [ddim_views][3][H][W], fp32 (reading A25)
 *    Ray id r = (v*H + i)*W + j; sample id = r*N + k.
 *  - Alignment: every tensor pointer must be 16-byte aligned
 *    (DMV3D_ERR_ALIGNMENT otherwise).
 */
#ifndef DMV3D_H
#define DMV3D_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *dmv3d_stream; /* == cudaStream_t */

typedef enum {
  DMV3D_OK = 0,
  DMV3D_ERR_INVALID_ARG = 1, /* a value outside its documented range            */
  DMV3D_ERR_UNSUPPORTED = 2, /* valid, but no kernel variant for this shape     */
  DMV3D_ERR_CUDA = 3,        /* a CUDA runtime call / launch failed             */
  DMV3D_ERR_ALIGNMENT = 4    /* a tensor pointer is not 16-byte aligned         */
} dmv3d_status;

/* FP8_E4M3: triplane storage only (row f4), value = fp8_scale * e4m3 (OCP E4M3,
 * finite range +-448), TCGEN05 engine only (its pre-projection decodes it). */
typedef enum { DMV3D_F32 = 0, DMV3D_BF16 = 1, DMV3D_FP8_E4M3 = 2 } dmv3d_dtype;
/* A4; CONCAT (row f4) feeds [f_XY, f_XZ, f_YZ] (in_dim = 3 C) to the MLP */
typedef enum { DMV3D_AGG_MEAN = 0, DMV3D_AGG_SUM = 1, DMV3D_AGG_CONCAT = 2 } dmv3d_agg;
/* Texel addressing (A3).  ALIGN_CORNERS: texel centres at the box faces, clamped
 * (grid_sample align_corners=True, border); HALFPIXEL_ZEROS (row f4): centres at
 * (i + 1/2)/R of the box, corners outside the plane read as zero
 * (grid_sample align_corners=False, padding zeros). */
typedef enum { DMV3D_SAMPLE_ALIGN_CORNERS = 0, DMV3D_SAMPLE_HALFPIXEL_ZEROS = 1 } dmv3d_sample_mode;
typedef enum { DMV3D_ACT_RELU = 0, DMV3D_ACT_SILU = 1, DMV3D_ACT_SOFTPLUS = 2 } dmv3d_act;
typedef enum {
  DMV3D_ENGINE_AUTO = 0,   /* tensor cores when the shapes allow, else SIMT            */
  DMV3D_ENGINE_SIMT = 1,   /* fp32 CUDA-core MLP (fp32 or bf16 storage)                */
  DMV3D_ENGINE_TCGEN05 = 2 /* tensor cores: bf16 storage, blend + MLP as fp16 tcgen05
                              MMAs with fp32 TMEM accumulation; hidden 64 (ReLU, SiLU or
                              softplus hidden layers; the backward: ReLU), needs
                              opts.workspace.  Projected triplane and activations are
                              fp16: a value beyond +-65504 is NOT clamped, it becomes
                              inf / NaN in the outputs and raises the call's range flag
                              (dmv3d_range_flags)                                       */
} dmv3d_engine;

/* Camera set C ("viewpoints C = {c_1..c_N}"). */
typedef struct {
  int32_t num_views, height, width; /* V, H, W >= 1                              */
  const float *intrinsics;          /* [V][4]    DEVICE                           */
  const float *c2w;                 /* [V][3][4] DEVICE                           */
} dmv3d_cameras;

/* Triplane S_t (reading A1: R = 64, C = 32 or 80). */
typedef struct {
  int32_t res, channels; /* R >= 2; C >= 1 (C % 4 == 0 for F32, C % 8 == 0 for BF16,
                            C % 16 == 0 for FP8_E4M3)                              */
  dmv3d_dtype dtype;
  const void *data;      /* [3][R][R][C] DEVICE                                   */
  float aabb_min[3], aabb_max[3]; /* object box, default -1/+1    */
  dmv3d_sample_mode sample_mode;  /* texel addressing, default ALIGN_CORNERS         */
  float fp8_scale;       /* FP8_E4M3 dequantisation scale (0 is read as 1); ignored
                            for the other dtypes                                    */
} dmv3d_triplane;

/* Shared MLP decoder (reading A5-A7).  Layer l maps
 * in_l -> out_l with in_0 = in_dim (= channels; 3 * channels for CONCAT), out_{L-1} = 4 (sigma, r, g, b),
 * every other width = hidden.  sigma = softplus(o_0 + density_shift);
 * c = sigmoid(o_{1..3}) * (1 + 2 eps) - eps. */
typedef struct {
  int32_t num_layers, in_dim, hidden; /* 2 <= L <= 8                                */
  dmv3d_dtype dtype;                  /* weight storage; biases are always fp32     */
  const void *const *weights;         /* HOST array of L DEVICE pointers, W_l [out][in] */
  const float *const *biases;         /* HOST array of L DEVICE pointers, b_l [out]     */
  dmv3d_act hidden_act;
  float density_shift, rgb_widen_eps;
} dmv3d_mlp;

/* Ray-marching options (readings A9-A14). */
typedef struct {
  int32_t samples_per_ray; /* N, 1 <= N <= 1024 (BASELINE: 128)                       */
  dmv3d_agg agg;
  int32_t jitter;          /* 0: midpoints; 1: stratified, splitmix64(seed, r*N+k)      */
  uint64_t seed;
  float bg_rgb[3];         /* background, default white                 */
  float term_eps;          /* early ray termination when T < term_eps; 0 disables.
                              |rgb - rgb_full|, |A - A_full| <= term_eps (A14)         */
  int64_t ray_begin, ray_end; /* shard [begin, end) of global ray ids; -1,-1 = all.
                              Only pixels of the shard are written.                    */
  dmv3d_engine engine;
  unsigned long long *counters; /* optional DEVICE [8] accumulators (NULL = off):
                              [0] rays hit, [1] samples evaluated,
                              [2] rays terminated early, [3] rays processed,
                              TCGEN05 only: [4] tensor-core tile rows issued (128 per
                              blend window: evaluated / issued = MMA row occupancy),
                              [5] staged texel columns (K) summed over blend windows,
                              [6] evaluated samples whose head output was not finite
                              (fp16 overflow upstream, see dmv3d_range_flags),
                              [7] reserved (0)                                         */
  void *workspace;         /* DEVICE scratch of >= dmv3d_workspace_bytes() bytes, 256-B
                              aligned; required by the TCGEN05 engine (holds the
                              per-step projected triplane), ignored by SIMT.  One
                              workspace per stream: calls sharing it must be ordered. */
  uint64_t workspace_bytes;
  struct dmv3d_timer *timer; /* optional: CUDA events are recorded around the render
                              kernel of this call (see dmv3d_timer_*); NULL = off     */
  float *plucker;          /* optional DEVICE [V][6][H][W]: the Plucker ray map
                              (o x d, d) of every rendered pixel,
                              written during ray generation; NULL = off              */
  int32_t num_peers;       /* 0..7.  Every rgb / alpha / x_prev value this launch
                              writes is also stored, at the same element offset, into
                              each peer buffer below: P2P stores over NVLink into
                              peer-mapped (e.g. symmetric-memory) buffers, so a view-
                              sharded step assembles the full outputs on every GPU from
                              the render epilogue itself (no separate all-gather).  The
                              caller orders the peers' reads after this launch (a
                              cross-GPU barrier).                                     */
  float *const *peer_rgb;  /* HOST array [num_peers] of DEVICE pointers laid out like
                              the rgb argument (NULL entry: skip that peer); same for
                              alpha and x_prev.  The arrays may be NULL when unused.  */
  float *const *peer_alpha;
  float *const *peer_x_prev;
  int32_t tile_size;       /* interleaved ray tiles, render / DDIM calls:
                              0 = off; else T > 0 (a multiple of 4) and only the pixels
                              of tiles tau = (v ceil(H/T) + i/T) ceil(W/T) + j/T with
                              tau mod tile_count == tile_rank are rendered and written
                              (the others are left untouched).  Balances AABB misses and
                              early termination across ranks.                          */
  int32_t tile_rank, tile_count;
  const float *fwd_rgb;    /* backward only, optional DEVICE [V][3][H][W] / [V][H][W]: the  */
  const float *fwd_alpha;  /* forward render of the same call (rgb, alpha; term_eps 0, or
                              within term_eps).  Given both, the backward takes C = rgb
                              and T_N = 1 - alpha from them instead of marching every
                              ray a first time (training has them from its forward).  */
} dmv3d_render_opts;

/* Launch timer for measurement: each render call with opts.timer set records
 * one (start, end) CUDA-event pair on its stream around the dominant render
 * kernel (the TCGEN05 pre-projection launch is outside the bracket).
 * dmv3d_timer_read synchronises on the recorded events and returns the summed
 * device time and the number of bracketed launches since the last reset. */
typedef struct dmv3d_timer dmv3d_timer;
dmv3d_status dmv3d_timer_create(dmv3d_timer **timer);
dmv3d_status dmv3d_timer_destroy(dmv3d_timer *timer);
dmv3d_status dmv3d_timer_reset(dmv3d_timer *timer);
dmv3d_status dmv3d_timer_read(dmv3d_timer *timer, double *total_ms, int64_t *launches);

/* Scratch the TCGEN05 engine needs for this triplane/MLP (0 if it cannot run
 * them), enough for every TCGEN05 call: a 256-B header, the projected triplane
 * G [(3*R*R + 1)][hidden] fp16 (the extra row holds b0) and, 256-B aligned after
 * it, the backward's projected-space gradient dG [(3*R*R + 1)][hidden] fp32.
 * Rendering alone needs only 256 + (3*R*R + 1)*hidden*2 bytes. */
uint64_t dmv3d_workspace_bytes(const dmv3d_triplane *triplane, const dmv3d_mlp *mlp);

/* fp16 range guard of the TCGEN05 engine (the projected triplane G = F W0^T + b0 and the
 * hidden activations are fp16 MMA operands).  Reads the range flags of the last
 * TCGEN05 call that used `workspace` (enqueued on `stream`; this call synchronises the
 * stream): bit 0 = some G value was outside +-65504 (or NaN), bit 1 = some evaluated
 * sample's head output was not finite (an activation overflowed fp16; a weight of
 * layers 1..L-1 beyond +-65504 becomes inf in its fp16 copy and shows up here too;
 * weights below fp16's smallest subnormal, 6e-8, round to 0).  Either bit
 * means the call's outputs contain inf / NaN: rescale the triplane / weights or use
 * the SIMT engine (fp32).  0 = in range.  The flags are cleared by every call that
 * projects the triplane (each TCGEN05 render / DDIM / backward / grid call). */
#define DMV3D_RANGE_G_OVERFLOW 1u
#define DMV3D_RANGE_ACT_OVERFLOW 2u
dmv3d_status dmv3d_range_flags(const void *workspace, uint32_t *flags, dmv3d_stream stream);

/* The engine a render / DDIM call with these arguments runs (AUTO resolved): writes
 * DMV3D_ENGINE_SIMT or DMV3D_ENGINE_TCGEN05 to *engine, or returns the status the call
 * would fail with.  AUTO takes the tensor cores whenever they can run the call (bf16
 * triplane + weights, hidden 64, a workspace) and otherwise the fp32 SIMT engine, which
 * is ~20x slower at cfg3: callers that need the fast path check it here.  No device
 * work. */
dmv3d_status dmv3d_select_engine(const dmv3d_triplane *triplane, const dmv3d_mlp *mlp,
                                 const dmv3d_render_opts *opts, int32_t num_assets,
                                 dmv3d_engine *engine);

/* DDIM x0 -> x_{t-1} (readings A15-A20). */
typedef struct {
  const double *alpha_bar; /* HOST [T], 0-based alpha_bar_t in (0,1], decreasing    */
  int32_t T, t, t_prev;    /* 0 <= t < T, -1 <= t_prev < t (t_prev = -1: ab_p = 1)   */
  float eta;               /* [0,1]; eta > 0 needs z                                */
  float x0_scale, x0_shift;/* x0_hat = scale * rgb + shift (default 2, -1)           */
  const uint8_t *keep_mask;/* HOST [ddim_views] or NULL: 1 = view kept noise-free,
                              x_{t-1} = x_t (image conditioning)        */
  int32_t ddim_views;      /* views [0, ddim_views) of the camera set get the update;
                              1 <= ddim_views <= min(V, 64)                          */
  int32_t noise_in_kernel; /* eta > 0 and z == NULL: draw z in the kernel (row f4):
                              element e of x_t gets Box-Muller of splitmix64(seed,
                              2e+1), splitmix64(seed, 2e+2) (24-bit uniforms)        */
  uint64_t noise_seed;
  int32_t skip_kept_views; /* fused steps: 1 = views with keep_mask set are NOT rendered
                              (their rgb / alpha are left untouched; x_{t-1} = x_t is
                              written); 0 = they are rendered like any other view     */
} dmv3d_ddim_params;

/* ---------------------------------------------------------------- renderer */
/* R(S, c) for every view of `cams`: rgb [V][3][H][W] (required), alpha
 * [V][H][W] (NULL = not written). */
dmv3d_status dmv3d_render_views(const dmv3d_triplane *triplane, const dmv3d_cameras *cams,
                                const dmv3d_mlp *mlp, const dmv3d_render_opts *opts,
                                float *rgb, float *alpha, dmv3d_stream stream);

/* Standalone DDIM step over [V][3][H][W]: x_prev from x_t and the rendered x0
 * image x0_rgb.  z may be NULL iff eta == 0.  params->ddim_views is ignored
 * (V is given); keep_mask, when set, has V entries. */
dmv3d_status dmv3d_ddim_step(const dmv3d_ddim_params *params, int32_t V, int32_t H, int32_t W,
                             const float *x_t, const float *x0_rgb, const float *z,
                             float *x_prev, dmv3d_stream stream);

/* One denoising step, fused: render all views of `cams` and, for the first
 * ddim_views views, apply the DDIM update in the per-ray epilogue.
 * x_t, z (NULL iff eta == 0), x_prev: [ddim_views][3][H][W].
 * rgb [V][3][H][W] and alpha [V][H][W] may each be NULL; when BOTH are NULL only the
 * views [0, ddim_views) are rendered (the others have no output to write). */
dmv3d_status dmv3d_render_ddim_step(const dmv3d_triplane *triplane, const dmv3d_cameras *cams,
                                    const dmv3d_mlp *mlp, const dmv3d_render_opts *opts,
                                    const dmv3d_ddim_params *ddim, const float *x_t,
                                    const float *z, float *x_prev, float *rgb, float *alpha,
                                    dmv3d_stream stream);

/* Batched assets (cfg4: PAPER.md:2538 trains/samples with 8 assets per GPU): one
 * launch renders num_assets assets that share the MLP and (V, H, W), assets as the
 * outer dimension of the work queue.  Every per-asset tensor gains a leading asset
 * dimension, contiguous: triplane->data [A][3][R][R][C], cams->intrinsics [A][V][4],
 * cams->c2w [A][V][3][4] (cams->num_views = V per asset), rgb [A][V][3][H][W], alpha
 * [A][V][H][W], x_t / z / x_prev [A][ddim_views][3][H][W]; keep_mask [ddim_views]
 * applies to every asset; opts ray ranges and tiles count global views a*V + v (ray
 * id r = ((a V + v) H + i) W + j), and in-kernel noise uses the element index of the
 * batched x_t.  The TCGEN05 engine needs dmv3d_workspace_bytes_batched() bytes (one
 * projected triplane per asset).  Bitwise equal, asset by asset, to single-asset calls. */
dmv3d_status dmv3d_render_views_batched(const dmv3d_triplane *triplane, int32_t num_assets,
                                        const dmv3d_cameras *cams, const dmv3d_mlp *mlp,
                                        const dmv3d_render_opts *opts, float *rgb, float *alpha,
                                        dmv3d_stream stream);
dmv3d_status dmv3d_render_ddim_step_batched(const dmv3d_triplane *triplane, int32_t num_assets,
                                            const dmv3d_cameras *cams, const dmv3d_mlp *mlp,
                                            const dmv3d_render_opts *opts,
                                            const dmv3d_ddim_params *ddim, const float *x_t,
                                            const float *z, float *x_prev, float *rgb,
                                            float *alpha, dmv3d_stream stream);
/* Render-only scratch of the TCGEN05 engine for num_assets assets (0 if it cannot run
 * them); num_assets == 1 returns dmv3d_workspace_bytes(). */
uint64_t dmv3d_workspace_bytes_batched(const dmv3d_triplane *triplane, const dmv3d_mlp *mlp,
                                       int32_t num_assets);

/* Plucker ray map: r = (o x d, d) per pixel, "concatenated with
 * image pixels" as the denoiser's camera conditioning, with o,
 * d the same bit-exact fp32 rays the renderer marches.  out [V][6][H][W]
 * (channels m_x, m_y, m_z, d_x, d_y, d_z); opts may be NULL (all rays) or give
 * a ray range. */
dmv3d_status dmv3d_plucker_rays(const dmv3d_cameras *cams, const dmv3d_render_opts *opts,
                                float *out, dmv3d_stream stream);

/* Renderer backward: the gradient of
 *   L = sum grad_rgb * rgb + sum grad_alpha * alpha
 * w.r.t. the triplane and the MLP parameters, through the same rays, samples,
 * gather, MLP and quadrature as dmv3d_render_views -- the "differentiable volume
 * rendering" L_recon trains through.  opts.term_eps > 0
 * differentiates the early-terminated render (the forward engines' rule: a ray stops
 * after the chunk where T < term_eps; later samples get no gradient); 0 = the full
 * quadrature.  grad_rgb [V][3][H][W], grad_alpha [V][H][W] or
 * NULL; outputs are fp32 and ACCUMULATED (caller zeroes them): grad_triplane
 * [3][R][R][C], grad_weights / grad_biases = HOST arrays of L DEVICE pointers
 * shaped like W_l / b_l.  ReLU hidden layers only; atomics make the summation
 * order, hence the last bits, run-dependent.
 * Engines: SIMT = fp32 CUDA cores (any supported shape).  TCGEN05 (also taken by
 * AUTO when opts.workspace holds dmv3d_workspace_bytes()): bf16 triplane and
 * weights, hidden 64, 2 <= L <= 7; the gradient of the first layer is accumulated
 * in the projected space (dG = A^T dz0 on the tensor cores, then dF = dG W0,
 * dW0 = dG^T F), activations and deltas are fp16 MMA operands with fp32
 * accumulation.  The workspace is overwritten. */
dmv3d_status dmv3d_render_backward(const dmv3d_triplane *triplane, const dmv3d_cameras *cams,
                                   const dmv3d_mlp *mlp, const dmv3d_render_opts *opts,
                                   const float *grad_rgb, const float *grad_alpha,
                                   float *grad_triplane, float *const *grad_weights,
                                   float *const *grad_biases, dmv3d_stream stream);

/* Density grid: sigma (and rgb) of the shared MLP decoder at the
 * G^3 points p_a = lo_a + (i_a/(G-1)) (hi_a - lo_a) of the triplane's box, the
 * input of marching cubes for the paper's Chamfer-distance evaluation and mesh
 * extraction.  sigma [G][G][G] and rgb [3][G][G][G] (NULL = not
 * written), x fastest; 2 <= grid_res <= 2048.  From `opts` (NULL = SIMT, mean)
 * only agg, engine, workspace and timer are read: the TCGEN05 engine decodes
 * 8x4x4 blocks of points through the same staged-texel blend + MLP MMAs as the
 * renderer (needs the workspace), SIMT in fp32. */
dmv3d_status dmv3d_density_grid(const dmv3d_triplane *triplane, const dmv3d_mlp *mlp,
                                const dmv3d_render_opts *opts, int32_t grid_res, float *sigma,
                                float *rgb, dmv3d_stream stream);

/* ------------------------------------------------------ host-buffer variant */
/* Same step with every tensor pointer (triplane data, weights, biases,
 * intrinsics, c2w, x_t, z, x_prev, rgb, alpha) a HOST pointer (pinned for
 * async copies).  The workspace owns grow-only device buffers, a copy stream and
 * events; one workspace per thread/stream.  Copies in on `stream`, then the views
 * are rendered in up to 2 view chunks (ray ranges; bitwise the same result as one
 * launch) and each chunk's outputs are copied out on the workspace's copy stream
 * while the next chunk renders; `stream` waits for the last copy, so the host
 * buffers are valid after `stream` is synchronised. */
typedef struct dmv3d_workspace dmv3d_workspace;
dmv3d_status dmv3d_workspace_create(dmv3d_workspace **ws);
dmv3d_status dmv3d_workspace_destroy(dmv3d_workspace *ws);
/* Range flags (see dmv3d_range_flags) of the last host-buffer step run with `ws`;
 * synchronises the workspace's device. */
dmv3d_status dmv3d_workspace_range_flags(dmv3d_workspace *ws, uint32_t *flags);
dmv3d_status dmv3d_render_ddim_step_host(dmv3d_workspace *ws, const dmv3d_triplane *triplane,
                                         const dmv3d_cameras *cams, const dmv3d_mlp *mlp,
                                         const dmv3d_render_opts *opts,
                                         const dmv3d_ddim_params *ddim, const float *x_t,
                                         const float *z, float *x_prev, float *rgb,
                                         float *alpha, dmv3d_stream stream);

/* Interleaved-tile merge (opts.tile_size / tile_rank / tile_count).  Packed
 * layout: rank r's k-th tile (tile id tau = r + k world over the whole camera set, the
 * ids of the tile formula above) is block k of that rank's rgb [nmax][3][T][T], alpha
 * [nmax][T][T] and x_prev [nmax][3][T][T], nmax = ceil(tiles / world) (a rank's blocks
 * past its last tile are unused; x_prev blocks only for views < ddim_views).
 * dmv3d_tiles_pack copies rank `rank`'s tiles from image-layout rgb [V][3][H][W], alpha
 * [V][H][W], x_prev [ddim_views][3][H][W] (a tile-sharded render's outputs) into its
 * blocks; after the ranks' blocks are all-gathered back to back ([world][nmax]...),
 * dmv3d_tiles_unpack scatters every rank's blocks into the images.  Any of the three
 * (image, packed) pairs may be NULL.  Async on `stream`; one HBM-bound pass each. */
dmv3d_status dmv3d_tiles_pack(const dmv3d_cameras *cams, int32_t tile_size, int32_t rank, int32_t world,
                              int32_t ddim_views, const float *rgb, const float *alpha,
                              const float *x_prev, float *packed_rgb, float *packed_alpha,
                              float *packed_x_prev, dmv3d_stream stream);
dmv3d_status dmv3d_tiles_unpack(const dmv3d_cameras *cams, int32_t tile_size, int32_t world,
                                int32_t ddim_views, const float *packed_rgb,
                                const float *packed_alpha, const float *packed_x_prev,
                                float *rgb, float *alpha, float *x_prev, dmv3d_stream stream);

/* Thread-local message describing the last non-OK status ("" if none). */
const char *dmv3d_last_error(void);
/* Library version string. */
const char *dmv3d_version(void);

/* ----------------------------------------------- stage-level entry points */
/* Bit-exact geometry for rays [ray_begin, ray_end) of opts (all when -1):
 * o_d [n][6] (origin, unit direction), tn_tf [n][2], hit [n] (0/1).  Misses
 * report t_near = t_far = 0.  Any output may be NULL. */
dmv3d_status dmv3d_debug_ray_geometry(const dmv3d_cameras *cams, const float aabb_min[3],
                                      const float aabb_max[3], const dmv3d_render_opts *opts,
                                      float *o_d, float *tn_tf, uint8_t *hit,
                                      dmv3d_stream stream);
/* Bit-exact sample set: t_k [n][N], point [n][N][3], texel [n][N][3][2]
 * (column, row index per plane), frac [n][N][3][2] (fractions); rays that
 * miss write zeros.  Only res, aabb and sample_mode of `grid` are read (its data
 * may be NULL).  HALFPIXEL_ZEROS reports the unclamped lower texel index
 * (-1 .. R-1) and its fraction.  Any output may be NULL. */
dmv3d_status dmv3d_debug_sample_points(const dmv3d_cameras *cams, const dmv3d_triplane *grid,
                                       const dmv3d_render_opts *opts,
                                       float *t_k, float *points, int32_t *texel, float *frac,
                                       dmv3d_stream stream);
/* Aggregated triplane features at n points [n][3] -> feats [n][C] ([n][3C] for
 * CONCAT) (fp32 math). */
dmv3d_status dmv3d_debug_sample_features(const dmv3d_triplane *triplane, dmv3d_agg agg,
                                         int64_t n, const float *points, float *feats,
                                         dmv3d_stream stream);
/* Gather + MLP decode at n points -> sigma_rgb [n][4] (engine SIMT, fp32 math). */
dmv3d_status dmv3d_debug_decode(const dmv3d_triplane *triplane, const dmv3d_mlp *mlp,
                                dmv3d_agg agg, int64_t n, const float *points,
                                float *sigma_rgb, dmv3d_stream stream);

#ifdef __cplusplus
}
#endif
#endif /* DMV3D_H */
