// api.cu -- the C ABI of libdmv3d.so (include/dmv3d.h): argument validation,
// launch-parameter marshalling, engine dispatch, the host-buffer workspace.
// No torch types; no device allocation on the device-pointer entry points.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <string.h>

#include <string>
#include <vector>

#include "../../include/dmv3d.h"
#include "common.cuh"
#include "kernels.h"

using namespace dmv3d;

// Launch timer: a pool of CUDA event pairs recorded around each render kernel.
struct dmv3d_timer {
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
  size_t used = 0;
};

namespace dmv3d {
void timer_begin(void *t, cudaStream_t st) {
  if (!t) return;
  auto *tm = static_cast<dmv3d_timer *>(t);
  if (tm->used == tm->ev.size()) {
    cudaEvent_t a, b;
    if (cudaEventCreate(&a) != cudaSuccess) return;
    if (cudaEventCreate(&b) != cudaSuccess) {
      cudaEventDestroy(a);
      return;
    }
    tm->ev.emplace_back(a, b);
  }
  cudaEventRecord(tm->ev[tm->used].first, st);
}
void timer_end(void *t, cudaStream_t st) {
  if (!t) return;
  auto *tm = static_cast<dmv3d_timer *>(t);
  if (tm->used < tm->ev.size()) cudaEventRecord(tm->ev[tm->used++].second, st);
}
}  // namespace dmv3d

namespace {

thread_local std::string g_err;

dmv3d_status fail(dmv3d_status s, const std::string &msg) {
  g_err = msg;
  return s;
}

bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

#define CHECK_ARG(cond, msg) \
  do {                       \
    if (!(cond)) return fail(DMV3D_ERR_INVALID_ARG, msg); \
  } while (0)
#define CHECK_ALIGN(p, name) \
  do {                       \
    if (!aligned16(p)) return fail(DMV3D_ERR_ALIGNMENT, std::string(name) + " is not 16-byte aligned"); \
  } while (0)

dmv3d_status check_cams(const dmv3d_cameras *c) {
  CHECK_ARG(c != nullptr, "cameras is NULL");
  CHECK_ARG(c->num_views >= 1 && c->height >= 1 && c->width >= 1, "cameras: V, H, W must be >= 1");
  CHECK_ARG((int64_t)c->num_views * c->height * c->width < (int64_t(1) << 40), "cameras: too many rays");
  CHECK_ARG(c->intrinsics && c->c2w, "cameras: intrinsics / c2w is NULL");
  CHECK_ALIGN(c->intrinsics, "cameras.intrinsics");
  CHECK_ALIGN(c->c2w, "cameras.c2w");
  return DMV3D_OK;
}

dmv3d_status check_aabb(const float lo[3], const float hi[3]) {
  for (int a = 0; a < 3; ++a)
    CHECK_ARG(isfinite(lo[a]) && isfinite(hi[a]) && hi[a] > lo[a], "aabb: need finite lo < hi");
  return DMV3D_OK;
}

dmv3d_status check_triplane(const dmv3d_triplane *t) {
  CHECK_ARG(t != nullptr, "triplane is NULL");
  CHECK_ARG(t->res >= 2 && t->res <= 8192, "triplane: res must be in [2, 8192]");
  CHECK_ARG(t->channels >= 1, "triplane: channels must be >= 1");
  CHECK_ARG(t->dtype == DMV3D_F32 || t->dtype == DMV3D_BF16 || t->dtype == DMV3D_FP8_E4M3,
            "triplane: bad dtype");
  CHECK_ARG(isfinite(t->fp8_scale), "triplane: non-finite fp8_scale");
  CHECK_ARG(t->data != nullptr, "triplane: data is NULL");
  CHECK_ALIGN(t->data, "triplane.data");
  CHECK_ARG(t->sample_mode == DMV3D_SAMPLE_ALIGN_CORNERS || t->sample_mode == DMV3D_SAMPLE_HALFPIXEL_ZEROS,
            "triplane: bad sample_mode");
  if (t->dtype == DMV3D_F32 && t->channels % 4)
    return fail(DMV3D_ERR_UNSUPPORTED, "triplane: fp32 needs channels % 4 == 0 (16-byte vectors)");
  if (t->dtype == DMV3D_BF16 && t->channels % 8)
    return fail(DMV3D_ERR_UNSUPPORTED, "triplane: bf16 needs channels % 8 == 0 (16-byte vectors)");
  if (t->dtype == DMV3D_FP8_E4M3 && t->channels % 16)
    return fail(DMV3D_ERR_UNSUPPORTED, "triplane: fp8 needs channels % 16 == 0 (16-byte vectors)");
  return check_aabb(t->aabb_min, t->aabb_max);
}

dmv3d_status check_agg(int agg) {
  CHECK_ARG(agg == DMV3D_AGG_MEAN || agg == DMV3D_AGG_SUM || agg == DMV3D_AGG_CONCAT, "bad agg");
  return DMV3D_OK;
}

dmv3d_status check_mlp(const dmv3d_mlp *m, const dmv3d_triplane *t, int agg) {
  CHECK_ARG(m != nullptr, "mlp is NULL");
  CHECK_ARG(m->num_layers >= 2 && m->num_layers <= kMaxLayers, "mlp: num_layers must be in [2, 8]");
  if (agg == DMV3D_AGG_CONCAT)
    CHECK_ARG(m->in_dim == 3 * t->channels, "mlp: in_dim must be 3 * channels (concat aggregation)");
  else
    CHECK_ARG(m->in_dim == t->channels, "mlp: in_dim must equal triplane channels (mean/sum aggregation)");
  CHECK_ARG(m->hidden >= 1, "mlp: hidden must be >= 1");
  CHECK_ARG(m->dtype == DMV3D_F32 || m->dtype == DMV3D_BF16, "mlp: bad dtype");
  CHECK_ARG(m->hidden_act >= DMV3D_ACT_RELU && m->hidden_act <= DMV3D_ACT_SOFTPLUS, "mlp: bad hidden_act");
  CHECK_ARG(m->weights && m->biases, "mlp: weights / biases array is NULL");
  CHECK_ARG(isfinite(m->density_shift) && isfinite(m->rgb_widen_eps), "mlp: non-finite shift/eps");
  for (int l = 0; l < m->num_layers; ++l) {
    CHECK_ARG(m->weights[l] && m->biases[l], "mlp: a layer pointer is NULL");
    CHECK_ALIGN(m->weights[l], "mlp.weights[l]");
    CHECK_ALIGN(m->biases[l], "mlp.biases[l]");
  }
  return DMV3D_OK;
}

dmv3d_status check_opts(const dmv3d_render_opts *o, int64_t nrays) {
  CHECK_ARG(o != nullptr, "opts is NULL");
  CHECK_ARG(o->samples_per_ray >= 1 && o->samples_per_ray <= 1024, "opts: samples_per_ray must be in [1, 1024]");
  CHECK_ARG(o->agg == DMV3D_AGG_MEAN || o->agg == DMV3D_AGG_SUM || o->agg == DMV3D_AGG_CONCAT,
            "opts: bad agg");
  CHECK_ARG(o->term_eps >= 0.0f && o->term_eps < 1.0f, "opts: term_eps must be in [0, 1)");
  CHECK_ARG(o->engine >= DMV3D_ENGINE_AUTO && o->engine <= DMV3D_ENGINE_TCGEN05, "opts: bad engine");
  for (int c = 0; c < 3; ++c) CHECK_ARG(isfinite(o->bg_rgb[c]), "opts: non-finite bg");
  const bool all = o->ray_begin == -1 && o->ray_end == -1;
  CHECK_ARG(all || (o->ray_begin >= 0 && o->ray_begin <= o->ray_end && o->ray_end <= nrays),
            "opts: ray range must be -1,-1 or 0 <= begin <= end <= V*H*W");
  if (o->counters) CHECK_ALIGN(o->counters, "opts.counters");

  if (o->workspace && (reinterpret_cast<uintptr_t>(o->workspace) & 255u))
    return fail(DMV3D_ERR_ALIGNMENT, "opts.workspace is not 256-byte aligned");
  CHECK_ARG(o->num_peers >= 0 && o->num_peers <= kMaxPeers, "opts: num_peers must be in [0, 7]");
  CHECK_ARG(o->tile_size == 0 || (o->tile_size > 0 && o->tile_size % 4 == 0 && o->tile_count >= 1 &&
                                  o->tile_rank >= 0 && o->tile_rank < o->tile_count),
            "opts: tiles need tile_size % 4 == 0 and 0 <= tile_rank < tile_count");
  return DMV3D_OK;
}

void fill_common(RenderParams &P, const dmv3d_triplane *t, const dmv3d_cameras *c,
                 const dmv3d_mlp *m, const dmv3d_render_opts *o) {
  memset(&P, 0, sizeof(P));
  P.V = c->num_views;
  P.V_asset = c->num_views;
  P.H = c->height;
  P.W = c->width;
  P.intr = c->intrinsics;
  P.c2w = c->c2w;
  P.R = t->res;
  P.C = t->channels;
  P.tp = t->data;
  P.smode = t->sample_mode;
  P.tp_fp8 = t->dtype == DMV3D_FP8_E4M3 ? 1 : 0;
  P.tp_scale = (t->dtype == DMV3D_FP8_E4M3 && t->fp8_scale != 0.0f) ? t->fp8_scale : 1.0f;
  for (int a = 0; a < 3; ++a) {
    P.lo[a] = t->aabb_min[a];
    P.hi[a] = t->aabb_max[a];
    // exact reciprocal when the extent (as the kernels compute it, in fp32) is 2^k
    const float ext = P.hi[a] - P.lo[a];
    int e2 = 0;
    const float mant = frexpf(ext, &e2);
    P.inv_ext[a] = (mant == 0.5f && isnormal(ext) && isnormal(1.0f / ext)) ? 1.0f / ext : 0.0f;
  }
  if (m) {
    P.L = m->num_layers;
    P.K = m->in_dim;
    P.HD = m->hidden;
    for (int l = 0; l < m->num_layers; ++l) {
      P.w[l] = m->weights[l];
      P.b[l] = m->biases[l];
    }
    P.act = m->hidden_act;
    P.dshift = m->density_shift;
    P.weps = m->rgb_widen_eps;
  }
  if (o) {
    P.N = o->samples_per_ray;
    P.agg = o->agg;
    P.jitter = o->jitter ? 1 : 0;
    P.seed = o->seed;
    for (int ch = 0; ch < 3; ++ch) P.bg[ch] = o->bg_rgb[ch];
    P.term_eps = o->term_eps;
    const int64_t nrays = (int64_t)P.V * P.H * P.W;
    P.ray_begin = (o->ray_begin == -1 && o->ray_end == -1) ? 0 : o->ray_begin;
    P.ray_end = (o->ray_begin == -1 && o->ray_end == -1) ? nrays : o->ray_end;
    P.counters = o->counters;
    P.ws = o->workspace;
    P.ws_bytes = o->workspace_bytes;
    P.timer = o->timer;
    P.plucker = o->plucker;
    P.npeers = o->num_peers;
    P.tile_size = o->tile_size;
    P.tile_rank = o->tile_rank;
    P.tile_count = o->tile_count > 0 ? o->tile_count : 1;

    for (int k = 0; k < o->num_peers; ++k) {
      P.peer_rgb[k] = o->peer_rgb ? o->peer_rgb[k] : nullptr;
      P.peer_alpha[k] = o->peer_alpha ? o->peer_alpha[k] : nullptr;
      P.peer_xp[k] = o->peer_x_prev ? o->peer_x_prev[k] : nullptr;
    }
  }
}

dmv3d_status ddim_coefficients(const dmv3d_ddim_params *d, int32_t nviews, DdimCoef &c) {
  CHECK_ARG(d != nullptr, "ddim params is NULL");
  CHECK_ARG(d->alpha_bar != nullptr, "ddim: alpha_bar is NULL");
  CHECK_ARG(d->T >= 1 && d->t >= 0 && d->t < d->T, "ddim: need 0 <= t < T");
  CHECK_ARG(d->t_prev >= -1 && d->t_prev < d->t, "ddim: need -1 <= t_prev < t");
  CHECK_ARG(d->eta >= 0.0f && d->eta <= 1.0f, "ddim: eta must be in [0, 1]");
  CHECK_ARG(isfinite(d->x0_scale) && isfinite(d->x0_shift), "ddim: non-finite x0 scale/shift");
  const double ab_t = d->alpha_bar[d->t];
  const double ab_p = d->t_prev >= 0 ? d->alpha_bar[d->t_prev] : 1.0;
  CHECK_ARG(ab_t > 0.0 && ab_t < 1.0, "ddim: alpha_bar[t] must be in (0, 1)");
  CHECK_ARG(ab_p > 0.0 && ab_p <= 1.0 && ab_p >= ab_t, "ddim: need alpha_bar[t] <= alpha_bar[t_prev] <= 1");
  const double sigma = (double)d->eta * sqrt((1.0 - ab_p) / (1.0 - ab_t)) * sqrt(1.0 - ab_t / ab_p);
  double c2 = 1.0 - ab_p - sigma * sigma;
  if (c2 < 0.0) c2 = 0.0;
  c.x0_scale = d->x0_scale;
  c.x0_shift = d->x0_shift;
  c.sqrt_ab_t = (float)sqrt(ab_t);
  c.inv_sqrt_1m_ab_t = (float)(1.0 / sqrt(1.0 - ab_t));
  c.sqrt_ab_p = (float)sqrt(ab_p);
  c.c_eps = (float)sqrt(c2);
  c.sigma_t = (float)sigma;
  c.keep_bits = 0;
  c.noise_seed = d->noise_seed;
  if (d->keep_mask) {
    if (nviews > 64) return fail(DMV3D_ERR_UNSUPPORTED, "ddim: keep_mask supports at most 64 views");
    for (int v = 0; v < nviews; ++v)
      if (d->keep_mask[v]) c.keep_bits |= (1ull << v);
  }
  return DMV3D_OK;
}

enum class Engine { SIMT, TC };

dmv3d_status pick_engine(const dmv3d_triplane *t, const dmv3d_mlp *m, const dmv3d_render_opts *o,
                         Engine &e, int assets = 1) {
  const bool bf16 = (t->dtype == DMV3D_BF16 || t->dtype == DMV3D_FP8_E4M3) && m->dtype == DMV3D_BF16;
  const bool tc_ok = bf16 &&
                     tc_supported(t->channels, m->hidden, m->num_layers);
  const bool ws_ok = o->workspace && o->workspace_bytes >= tc_workspace_bytes(t->res, m->hidden, assets);
  if (o->engine == DMV3D_ENGINE_TCGEN05) {
    if (!tc_ok)
      return fail(DMV3D_ERR_UNSUPPORTED,
                  "engine TCGEN05 needs bf16 triplane + weights, hidden 64, channels % 8 == 0 "
                  "(<= 256), 2 <= L <= 8");
    if (!ws_ok)
      return fail(DMV3D_ERR_INVALID_ARG,
                  "engine TCGEN05 needs opts.workspace of dmv3d_workspace_bytes() bytes");
    e = Engine::TC;
    return DMV3D_OK;
  }
  if (o->engine == DMV3D_ENGINE_AUTO && tc_ok && ws_ok) {
    e = Engine::TC;
    return DMV3D_OK;
  }
  if (t->dtype == DMV3D_FP8_E4M3)
    return fail(DMV3D_ERR_UNSUPPORTED, "fp8 triplane storage needs engine TCGEN05 (bf16 weights, "
                                       "hidden 64, a workspace)");
  if (!simt_supported(m->in_dim, m->hidden, o->agg == DMV3D_AGG_CONCAT))
    return fail(DMV3D_ERR_UNSUPPORTED, "SIMT engine: unsupported (in_dim, hidden) = (" +
                                           std::to_string(m->in_dim) + ", " + std::to_string(m->hidden) + ")");
  e = Engine::SIMT;
  return DMV3D_OK;
}

dmv3d_status cuda_status(cudaError_t e, const char *what) {
  if (e == cudaSuccess) return DMV3D_OK;
  return fail(DMV3D_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

dmv3d_status render_impl(const dmv3d_triplane *t, const dmv3d_cameras *c, const dmv3d_mlp *m,
                         const dmv3d_render_opts *o, const dmv3d_ddim_params *d, const float *x_t,
                         const float *z, float *x_prev, float *rgb, float *alpha,
                         cudaStream_t st, bool reuse_g = false, int assets = 1) {
  dmv3d_status s;
  if ((s = check_cams(c)) != DMV3D_OK) return s;
  if ((s = check_triplane(t)) != DMV3D_OK) return s;
  CHECK_ARG(assets >= 1 && (int64_t)assets * c->num_views < (int64_t(1) << 31),
            "batched: need 1 <= num_assets and num_assets * V < 2^31");
  const int64_t nrays = (int64_t)assets * c->num_views * c->height * c->width;
  CHECK_ARG(nrays < (int64_t(1) << 40), "too many rays");
  if ((s = check_opts(o, nrays)) != DMV3D_OK) return s;
  if ((s = check_mlp(m, t, o->agg)) != DMV3D_OK) return s;
  if (rgb) CHECK_ALIGN(rgb, "rgb");
  if (alpha) CHECK_ALIGN(alpha, "alpha");
  RenderParams P;
  fill_common(P, t, c, m, o);
  P.V = assets * c->num_views;  // batched: assets x V views, asset-major
  P.ray_end = (o->ray_begin == -1 && o->ray_end == -1) ? nrays : o->ray_end;
  P.rgb = rgb;
  P.alpha = alpha;
  P.reuse_g = reuse_g ? 1 : 0;
  if (d) {
    CHECK_ARG(d->ddim_views >= 1 && d->ddim_views <= c->num_views, "ddim: need 1 <= ddim_views <= V");
    if (d->ddim_views > 64) return fail(DMV3D_ERR_UNSUPPORTED, "ddim: at most 64 DDIM views per call");
    DdimCoef k;
    if ((s = ddim_coefficients(d, d->ddim_views, k)) != DMV3D_OK) return s;
    CHECK_ARG(x_t && x_prev, "ddim: x_t / x_prev is NULL");
    CHECK_ARG(k.sigma_t == 0.0f || z != nullptr || d->noise_in_kernel,
              "ddim: eta > 0 needs z or noise_in_kernel");
    P.noise_seed = k.noise_seed;
    CHECK_ALIGN(x_t, "x_t");
    CHECK_ALIGN(x_prev, "x_prev");
    if (z) CHECK_ALIGN(z, "z");
    P.ddim_views = d->ddim_views;
    P.keep_bits = k.keep_bits;
    P.x_t = x_t;
    P.z = z;
    P.x_prev = x_prev;
    P.x0_scale = k.x0_scale;
    P.x0_shift = k.x0_shift;
    P.sqrt_ab_t = k.sqrt_ab_t;
    P.inv_sqrt_1m_ab_t = k.inv_sqrt_1m_ab_t;
    P.sqrt_ab_p = k.sqrt_ab_p;
    P.c_eps = k.c_eps;
    P.sigma_t = k.sigma_t;
    // rays nobody needs: views >= ddim_views when neither rgb nor alpha is asked for,
    // and (opt-in) kept conditioning views, whose x_{t-1} is x_t
    P.ddim_only = (rgb == nullptr && alpha == nullptr) ? 1 : 0;
    P.skip_kept = (d->skip_kept_views && k.keep_bits) ? 1 : 0;
  } else {
    CHECK_ARG(rgb != nullptr, "rgb is NULL");
  }
  Engine e;
  if ((s = pick_engine(t, m, o, e, assets)) != DMV3D_OK) return s;
  if (assets > 1 && e == Engine::SIMT && t->dtype == DMV3D_FP8_E4M3)
    return fail(DMV3D_ERR_UNSUPPORTED, "fp8 triplane storage needs engine TCGEN05");
  cudaError_t ce;
  if (e == Engine::TC)
    ce = launch_render_tc(P, st);
  else
    ce = launch_render_simt(P, t->dtype == DMV3D_BF16, m->dtype == DMV3D_BF16, st);
  return cuda_status(ce, "render launch");
}

}  // namespace

// =========================================================== exported ABI
extern "C" {

const char *dmv3d_last_error(void) { return g_err.c_str(); }
const char *dmv3d_version(void) { return "dmv3d-b200 0.3 (sm_100a)"; }

dmv3d_status dmv3d_plucker_rays(const dmv3d_cameras *cams, const dmv3d_render_opts *opts,
                                float *out, dmv3d_stream stream) {
  g_err.clear();
  dmv3d_status s;
  if ((s = check_cams(cams)) != DMV3D_OK) return s;
  CHECK_ARG(out != nullptr, "plucker: out is NULL");
  CHECK_ALIGN(out, "plucker out");
  dmv3d_render_opts o{};
  if (opts) {
    o = *opts;
  } else {
    o.samples_per_ray = 1;
    o.ray_begin = o.ray_end = -1;
  }
  if ((s = check_opts(&o, (int64_t)cams->num_views * cams->height * cams->width)) != DMV3D_OK)
    return s;
  dmv3d_triplane t{};
  t.res = 2;
  t.channels = 4;
  for (int a = 0; a < 3; ++a) {
    t.aabb_min[a] = -1.0f;
    t.aabb_max[a] = 1.0f;
  }
  RenderParams P;
  fill_common(P, &t, cams, nullptr, &o);
  return cuda_status(launch_plucker(P, out, reinterpret_cast<cudaStream_t>(stream)),
                     "plucker launch");
}

dmv3d_status dmv3d_render_backward(const dmv3d_triplane *triplane, const dmv3d_cameras *cams,
                                   const dmv3d_mlp *mlp, const dmv3d_render_opts *opts,
                                   const float *grad_rgb, const float *grad_alpha,
                                   float *grad_triplane, float *const *grad_weights,
                                   float *const *grad_biases, dmv3d_stream stream) {
  g_err.clear();
  dmv3d_status s;
  if ((s = check_cams(cams)) != DMV3D_OK) return s;
  if ((s = check_triplane(triplane)) != DMV3D_OK) return s;
  if ((s = check_opts(opts, (int64_t)cams->num_views * cams->height * cams->width)) != DMV3D_OK)
    return s;
  if ((s = check_mlp(mlp, triplane, opts->agg)) != DMV3D_OK) return s;
  CHECK_ARG(grad_rgb && grad_triplane && grad_weights && grad_biases, "backward: NULL gradient buffer");
  if (opts->tile_size)
    return fail(DMV3D_ERR_UNSUPPORTED, "backward: interleaved tiles are a render option (use ray ranges)");
  CHECK_ALIGN(grad_rgb, "grad_rgb");
  if (grad_alpha) CHECK_ALIGN(grad_alpha, "grad_alpha");
  CHECK_ALIGN(grad_triplane, "grad_triplane");
  if (mlp->hidden_act != DMV3D_ACT_RELU)
    return fail(DMV3D_ERR_UNSUPPORTED, "backward: ReLU hidden layers only");
  // engine: the tensor-core backward needs bf16 storage, the TC engine's shapes and a
  // workspace of dmv3d_workspace_bytes(); AUTO takes it when all hold
  const bool tc_ok = (triplane->dtype == DMV3D_BF16 || triplane->dtype == DMV3D_FP8_E4M3) &&
                     mlp->dtype == DMV3D_BF16 &&
                     tc_backward_supported(triplane->channels, mlp->hidden, mlp->num_layers);
  const bool ws_ok = opts->workspace &&
                     opts->workspace_bytes >= tc_backward_workspace_bytes(triplane->res, mlp->hidden);
  bool use_tc = false;
  if (opts->engine == DMV3D_ENGINE_TCGEN05) {
    if (!tc_ok)
      return fail(DMV3D_ERR_UNSUPPORTED,
                  "backward engine TCGEN05 needs bf16 triplane + weights, hidden 64, channels % 8 == 0 "
                  "(<= 256), 2 <= L <= 7");
    if (!ws_ok)
      return fail(DMV3D_ERR_INVALID_ARG,
                  "backward engine TCGEN05 needs opts.workspace of dmv3d_workspace_bytes() bytes");
    use_tc = true;
  } else if (opts->engine == DMV3D_ENGINE_AUTO && tc_ok && ws_ok) {
    use_tc = true;
  }
  if (!use_tc && triplane->dtype == DMV3D_FP8_E4M3)
    return fail(DMV3D_ERR_UNSUPPORTED, "backward: fp8 triplane storage needs engine TCGEN05");
  if (!use_tc &&
      !backward_supported(mlp->in_dim, mlp->hidden, mlp->num_layers, opts->agg == DMV3D_AGG_CONCAT))
    return fail(DMV3D_ERR_UNSUPPORTED, "backward: unsupported (in_dim, hidden, L)");
  RenderParams P;
  fill_common(P, triplane, cams, mlp, opts);
  GradParams G{};
  G.g_rgb = grad_rgb;
  G.g_alpha = grad_alpha;
  G.dF = grad_triplane;
  CHECK_ARG((opts->fwd_rgb == nullptr) == (opts->fwd_alpha == nullptr),
            "backward: give both opts.fwd_rgb and opts.fwd_alpha, or neither");
  if (opts->fwd_rgb) {
    CHECK_ALIGN(opts->fwd_rgb, "opts.fwd_rgb");
    CHECK_ALIGN(opts->fwd_alpha, "opts.fwd_alpha");
  }
  G.fwd_rgb = opts->fwd_rgb;
  G.fwd_alpha = opts->fwd_alpha;
  for (int l = 0; l < mlp->num_layers; ++l) {
    CHECK_ARG(grad_weights[l] && grad_biases[l], "backward: a gradient layer pointer is NULL");
    G.dW[l] = grad_weights[l];
    G.db[l] = grad_biases[l];
  }
  if (use_tc)
    return cuda_status(launch_render_backward_tc(P, G, reinterpret_cast<cudaStream_t>(stream)),
                       "backward (tcgen05) launch");
  return cuda_status(launch_render_backward(P, G, triplane->dtype == DMV3D_BF16,
                                            mlp->dtype == DMV3D_BF16,
                                            reinterpret_cast<cudaStream_t>(stream)),
                     "backward launch");
}

dmv3d_status dmv3d_density_grid(const dmv3d_triplane *triplane, const dmv3d_mlp *mlp,
                                const dmv3d_render_opts *opts, int32_t grid_res, float *sigma,
                                float *rgb, dmv3d_stream stream) {
  g_err.clear();
  dmv3d_status s;
  if ((s = check_triplane(triplane)) != DMV3D_OK) return s;
  dmv3d_render_opts o{};
  o.samples_per_ray = 1;
  o.ray_begin = o.ray_end = -1;
  o.engine = DMV3D_ENGINE_SIMT;
  if (opts) {
    o.agg = opts->agg;
    o.engine = opts->engine;
    o.workspace = opts->workspace;
    o.workspace_bytes = opts->workspace_bytes;
    o.timer = opts->timer;
  }
  if ((s = check_agg(o.agg)) != DMV3D_OK) return s;
  if ((s = check_mlp(mlp, triplane, o.agg)) != DMV3D_OK) return s;
  CHECK_ARG(o.engine >= DMV3D_ENGINE_AUTO && o.engine <= DMV3D_ENGINE_TCGEN05, "bad engine");
  CHECK_ARG(grid_res >= 2 && grid_res <= 2048, "density grid: grid_res must be in [2, 2048]");
  CHECK_ARG(sigma != nullptr, "density grid: sigma is NULL");
  CHECK_ALIGN(sigma, "sigma");
  if (rgb) CHECK_ALIGN(rgb, "rgb");
  if (o.workspace && (reinterpret_cast<uintptr_t>(o.workspace) & 255u))
    return fail(DMV3D_ERR_ALIGNMENT, "opts.workspace is not 256-byte aligned");
  dmv3d_cameras c{};
  c.num_views = c.height = c.width = 1;
  RenderParams P;
  fill_common(P, triplane, &c, mlp, &o);
  Engine e;
  if ((s = pick_engine(triplane, mlp, &o, e)) != DMV3D_OK) return s;
  if (e == Engine::TC) {
    P.grid_res = grid_res;
    P.grid_sigma = sigma;
    P.grid_rgb = rgb;
    return cuda_status(launch_render_tc(P, reinterpret_cast<cudaStream_t>(stream)),
                       "density grid launch");
  }
  if (!simt_supported(mlp->in_dim, mlp->hidden, o.agg == DMV3D_AGG_CONCAT))
    return fail(DMV3D_ERR_UNSUPPORTED, "density grid: unsupported (in_dim, hidden)");
  return cuda_status(launch_density_grid(P, triplane->dtype == DMV3D_BF16,
                                         mlp->dtype == DMV3D_BF16, grid_res, sigma, rgb,
                                         reinterpret_cast<cudaStream_t>(stream)),
                     "density grid launch");
}

dmv3d_status dmv3d_timer_create(dmv3d_timer **t) {
  g_err.clear();
  CHECK_ARG(t != nullptr, "timer is NULL");
  *t = new dmv3d_timer();
  return DMV3D_OK;
}

dmv3d_status dmv3d_timer_destroy(dmv3d_timer *t) {
  g_err.clear();
  if (!t) return DMV3D_OK;
  for (auto &p : t->ev) {
    cudaEventDestroy(p.first);
    cudaEventDestroy(p.second);
  }
  delete t;
  return DMV3D_OK;
}

dmv3d_status dmv3d_timer_reset(dmv3d_timer *t) {
  g_err.clear();
  CHECK_ARG(t != nullptr, "timer is NULL");
  t->used = 0;
  return DMV3D_OK;
}

dmv3d_status dmv3d_timer_read(dmv3d_timer *t, double *total_ms, int64_t *launches) {
  g_err.clear();
  CHECK_ARG(t && total_ms && launches, "NULL argument");
  double tot = 0.0;
  for (size_t i = 0; i < t->used; ++i) {
    cudaError_t e = cudaEventSynchronize(t->ev[i].second);
    if (e != cudaSuccess) return cuda_status(e, "timer");
    float ms = 0.0f;
    e = cudaEventElapsedTime(&ms, t->ev[i].first, t->ev[i].second);
    if (e != cudaSuccess) return cuda_status(e, "timer");
    tot += ms;
  }
  *total_ms = tot;
  *launches = (int64_t)t->used;
  return DMV3D_OK;
}

uint64_t dmv3d_workspace_bytes(const dmv3d_triplane *triplane, const dmv3d_mlp *mlp) {
  if (!triplane || !mlp || triplane->res < 2) return 0;
  if (!tc_supported(triplane->channels, mlp->hidden, mlp->num_layers)) return 0;
  // enough for every tensor-core call: render (G) and backward (G + dG)
  return tc_backward_workspace_bytes(triplane->res, mlp->hidden);
}

dmv3d_status dmv3d_render_views(const dmv3d_triplane *triplane, const dmv3d_cameras *cams,
                                const dmv3d_mlp *mlp, const dmv3d_render_opts *opts, float *rgb,
                                float *alpha, dmv3d_stream stream) {
  g_err.clear();
  return render_impl(triplane, cams, mlp, opts, nullptr, nullptr, nullptr, nullptr, rgb, alpha,
                     reinterpret_cast<cudaStream_t>(stream));
}

dmv3d_status dmv3d_render_ddim_step(const dmv3d_triplane *triplane, const dmv3d_cameras *cams,
                                    const dmv3d_mlp *mlp, const dmv3d_render_opts *opts,
                                    const dmv3d_ddim_params *ddim, const float *x_t,
                                    const float *z, float *x_prev, float *rgb, float *alpha,
                                    dmv3d_stream stream) {
  g_err.clear();
  if (!ddim) return fail(DMV3D_ERR_INVALID_ARG, "ddim params is NULL");
  return render_impl(triplane, cams, mlp, opts, ddim, x_t, z, x_prev, rgb, alpha,
                     reinterpret_cast<cudaStream_t>(stream));
}

dmv3d_status dmv3d_render_views_batched(const dmv3d_triplane *triplane, int32_t num_assets,
                                        const dmv3d_cameras *cams, const dmv3d_mlp *mlp,
                                        const dmv3d_render_opts *opts, float *rgb, float *alpha,
                                        dmv3d_stream stream) {
  g_err.clear();
  return render_impl(triplane, cams, mlp, opts, nullptr, nullptr, nullptr, nullptr, rgb, alpha,
                     reinterpret_cast<cudaStream_t>(stream), false, num_assets);
}

dmv3d_status dmv3d_render_ddim_step_batched(const dmv3d_triplane *triplane, int32_t num_assets,
                                            const dmv3d_cameras *cams, const dmv3d_mlp *mlp,
                                            const dmv3d_render_opts *opts,
                                            const dmv3d_ddim_params *ddim, const float *x_t,
                                            const float *z, float *x_prev, float *rgb,
                                            float *alpha, dmv3d_stream stream) {
  g_err.clear();
  if (!ddim) return fail(DMV3D_ERR_INVALID_ARG, "ddim params is NULL");
  return render_impl(triplane, cams, mlp, opts, ddim, x_t, z, x_prev, rgb, alpha,
                     reinterpret_cast<cudaStream_t>(stream), false, num_assets);
}

uint64_t dmv3d_workspace_bytes_batched(const dmv3d_triplane *triplane, const dmv3d_mlp *mlp,
                                       int32_t num_assets) {
  if (!triplane || !mlp || triplane->res < 2 || num_assets < 1) return 0;
  if (!tc_supported(triplane->channels, mlp->hidden, mlp->num_layers)) return 0;
  if (num_assets == 1) return dmv3d_workspace_bytes(triplane, mlp);
  return tc_workspace_bytes(triplane->res, mlp->hidden, num_assets);
}

dmv3d_status dmv3d_ddim_step(const dmv3d_ddim_params *params, int32_t V, int32_t H, int32_t W,
                             const float *x_t, const float *x0_rgb, const float *z, float *x_prev,
                             dmv3d_stream stream) {
  g_err.clear();
  CHECK_ARG(V >= 1 && H >= 1 && W >= 1, "ddim_step: V, H, W must be >= 1");
  DdimCoef k;
  dmv3d_status s = ddim_coefficients(params, V, k);
  if (s != DMV3D_OK) return s;
  CHECK_ARG(x_t && x0_rgb && x_prev, "ddim_step: x_t / x0_rgb / x_prev is NULL");
  CHECK_ARG(k.sigma_t == 0.0f || z != nullptr || params->noise_in_kernel,
            "ddim_step: eta > 0 needs z or noise_in_kernel");
  CHECK_ALIGN(x_t, "x_t");
  CHECK_ALIGN(x0_rgb, "x0_rgb");
  CHECK_ALIGN(x_prev, "x_prev");
  if (z) CHECK_ALIGN(z, "z");
  return cuda_status(launch_ddim(k, V, H, W, x_t, x0_rgb, z, nullptr, x_prev,
                                 reinterpret_cast<cudaStream_t>(stream)),
                     "ddim launch");
}

dmv3d_status dmv3d_debug_ray_geometry(const dmv3d_cameras *cams, const float aabb_min[3],
                                      const float aabb_max[3], const dmv3d_render_opts *opts,
                                      float *o_d, float *tn_tf, uint8_t *hit,
                                      dmv3d_stream stream) {
  g_err.clear();
  dmv3d_status s;
  if ((s = check_cams(cams)) != DMV3D_OK) return s;
  CHECK_ARG(aabb_min && aabb_max, "aabb is NULL");
  if ((s = check_aabb(aabb_min, aabb_max)) != DMV3D_OK) return s;
  if ((s = check_opts(opts, (int64_t)cams->num_views * cams->height * cams->width)) != DMV3D_OK)
    return s;
  dmv3d_triplane t{};
  t.res = 2;
  t.channels = 4;
  for (int a = 0; a < 3; ++a) {
    t.aabb_min[a] = aabb_min[a];
    t.aabb_max[a] = aabb_max[a];
  }
  RenderParams P;
  fill_common(P, &t, cams, nullptr, opts);
  return cuda_status(launch_ray_geometry(P, o_d, tn_tf, hit, reinterpret_cast<cudaStream_t>(stream)),
                     "ray geometry launch");
}

dmv3d_status dmv3d_debug_sample_points(const dmv3d_cameras *cams, const dmv3d_triplane *grid,
                                       const dmv3d_render_opts *opts, float *t_k, float *points,
                                       int32_t *texel, float *frac, dmv3d_stream stream) {
  g_err.clear();
  dmv3d_status s;
  if ((s = check_cams(cams)) != DMV3D_OK) return s;
  CHECK_ARG(grid != nullptr, "grid is NULL");
  CHECK_ARG(grid->res >= 2, "res must be >= 2");
  CHECK_ARG(grid->sample_mode == DMV3D_SAMPLE_ALIGN_CORNERS ||
                grid->sample_mode == DMV3D_SAMPLE_HALFPIXEL_ZEROS,
            "bad sample_mode");
  if ((s = check_aabb(grid->aabb_min, grid->aabb_max)) != DMV3D_OK) return s;
  if ((s = check_opts(opts, (int64_t)cams->num_views * cams->height * cams->width)) != DMV3D_OK)
    return s;
  dmv3d_triplane t = *grid;
  t.channels = 4;
  t.data = nullptr;
  RenderParams P;
  fill_common(P, &t, cams, nullptr, opts);
  return cuda_status(launch_sample_points(P, t_k, points, texel, frac,
                                          reinterpret_cast<cudaStream_t>(stream)),
                     "sample points launch");
}

static dmv3d_cameras no_cams() {
  dmv3d_cameras c{};
  c.num_views = c.height = c.width = 1;
  return c;
}

dmv3d_status dmv3d_debug_sample_features(const dmv3d_triplane *triplane, dmv3d_agg agg,
                                         int64_t n, const float *points, float *feats,
                                         dmv3d_stream stream) {
  g_err.clear();
  dmv3d_status s;
  if ((s = check_triplane(triplane)) != DMV3D_OK) return s;
  if ((s = check_agg(agg)) != DMV3D_OK) return s;
  CHECK_ARG(n >= 0, "n must be >= 0");
  CHECK_ARG(n == 0 || (points && feats), "points / feats is NULL");
  if (triplane->dtype == DMV3D_FP8_E4M3)
    return fail(DMV3D_ERR_UNSUPPORTED, "debug entry points are SIMT: no fp8 triplane storage");
  if (n) {
    CHECK_ALIGN(points, "points");
    CHECK_ALIGN(feats, "feats");
  }
  const dmv3d_cameras c = no_cams();
  RenderParams P;
  fill_common(P, triplane, &c, nullptr, nullptr);
  P.agg = agg;
  cudaError_t e = launch_features(P, triplane->dtype == DMV3D_BF16, n, points, feats,
                                  reinterpret_cast<cudaStream_t>(stream));
  if (e == cudaErrorInvalidValue)
    return fail(DMV3D_ERR_UNSUPPORTED, "features: unsupported channel count");
  return cuda_status(e, "features launch");
}

dmv3d_status dmv3d_debug_decode(const dmv3d_triplane *triplane, const dmv3d_mlp *mlp,
                                dmv3d_agg agg, int64_t n, const float *points, float *sigma_rgb,
                                dmv3d_stream stream) {
  g_err.clear();
  dmv3d_status s;
  if ((s = check_triplane(triplane)) != DMV3D_OK) return s;
  if ((s = check_agg(agg)) != DMV3D_OK) return s;
  if ((s = check_mlp(mlp, triplane, agg)) != DMV3D_OK) return s;
  CHECK_ARG(n >= 0, "n must be >= 0");
  CHECK_ARG(n == 0 || (points && sigma_rgb), "points / sigma_rgb is NULL");
  if (triplane->dtype == DMV3D_FP8_E4M3)
    return fail(DMV3D_ERR_UNSUPPORTED, "debug entry points are SIMT: no fp8 triplane storage");
  if (n) {
    CHECK_ALIGN(points, "points");
    CHECK_ALIGN(sigma_rgb, "sigma_rgb");
  }
  if (!simt_supported(mlp->in_dim, mlp->hidden, agg == DMV3D_AGG_CONCAT))
    return fail(DMV3D_ERR_UNSUPPORTED, "decode: unsupported (in_dim, hidden)");
  const dmv3d_cameras c = no_cams();
  RenderParams P;
  fill_common(P, triplane, &c, mlp, nullptr);
  P.agg = agg;
  return cuda_status(launch_decode(P, triplane->dtype == DMV3D_BF16, mlp->dtype == DMV3D_BF16, n,
                                   points, sigma_rgb, reinterpret_cast<cudaStream_t>(stream)),
                     "decode launch");
}

// ------------------------------------------------------ host-buffer variant
struct dmv3d_workspace {
  struct Buf {
    void *p = nullptr;
    size_t cap = 0;
  };
  Buf tp, intr, c2w, xt, z, xp, rgb, alpha, scratch, w[kMaxLayers], b[kMaxLayers];
  // copy-out pipeline: a stream for device->host copies and one event per view chunk
  static constexpr int kChunks = 2;
  cudaStream_t copy = nullptr;
  cudaEvent_t ev[kChunks + 1] = {};
  int dev = -1;
  const void *tc_ws = nullptr;  // the TCGEN05 workspace of the last step (range flags)
};

static cudaError_t ws_reserve(dmv3d_workspace::Buf &b, size_t bytes) {
  if (bytes <= b.cap) return cudaSuccess;
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
  b.cap = 0;
  cudaError_t e = cudaMalloc(&b.p, bytes);
  if (e == cudaSuccess) b.cap = bytes;
  return e;
}

dmv3d_status dmv3d_workspace_create(dmv3d_workspace **ws) {
  g_err.clear();
  CHECK_ARG(ws != nullptr, "ws is NULL");
  *ws = new dmv3d_workspace();
  return DMV3D_OK;
}

dmv3d_status dmv3d_workspace_destroy(dmv3d_workspace *ws) {
  g_err.clear();
  if (!ws) return DMV3D_OK;
  dmv3d_workspace::Buf *all[] = {&ws->tp, &ws->intr, &ws->c2w, &ws->xt, &ws->z,
                                 &ws->xp, &ws->rgb, &ws->alpha, &ws->scratch};
  for (auto *b : all)
    if (b->p) cudaFree(b->p);
  for (int l = 0; l < kMaxLayers; ++l) {
    if (ws->w[l].p) cudaFree(ws->w[l].p);
    if (ws->b[l].p) cudaFree(ws->b[l].p);
  }
  if (ws->copy) {
    cudaStreamDestroy(ws->copy);
    for (auto &ev : ws->ev) cudaEventDestroy(ev);
  }
  delete ws;
  return DMV3D_OK;
}

static dmv3d_status check_tiles(const dmv3d_cameras *cams, int32_t tile_size, int32_t world,
                                int32_t ddim_views, const float *a0, const float *a1, const float *b0,
                                const float *b1, const float *c0, const float *c1) {
  CHECK_ARG(cams != nullptr, "cameras is NULL");
  CHECK_ARG(cams->num_views >= 1 && cams->height >= 1 && cams->width >= 1, "cameras: V, H, W must be >= 1");
  CHECK_ARG(tile_size > 0 && tile_size % 4 == 0, "tiles: tile_size must be a positive multiple of 4");
  CHECK_ARG(world >= 1, "tiles: world must be >= 1");
  CHECK_ARG((a0 == nullptr) == (a1 == nullptr) && (b0 == nullptr) == (b1 == nullptr) &&
                (c0 == nullptr) == (c1 == nullptr),
            "tiles: packed / image buffers must be given in pairs");
  CHECK_ARG(c0 == nullptr || (ddim_views >= 1 && ddim_views <= cams->num_views),
            "tiles: need 1 <= ddim_views <= V for x_prev");
  return DMV3D_OK;
}

dmv3d_status dmv3d_tiles_pack(const dmv3d_cameras *cams, int32_t tile_size, int32_t rank, int32_t world,
                              int32_t ddim_views, const float *rgb, const float *alpha,
                              const float *x_prev, float *packed_rgb, float *packed_alpha,
                              float *packed_x_prev, dmv3d_stream stream) {
  g_err.clear();
  dmv3d_status s = check_tiles(cams, tile_size, world, ddim_views, rgb, packed_rgb, alpha, packed_alpha,
                               x_prev, packed_x_prev);
  if (s != DMV3D_OK) return s;
  CHECK_ARG(rank >= 0 && rank < world, "tiles_pack: need 0 <= rank < world");
  return cuda_status(launch_tiles_copy(cams->num_views, cams->height, cams->width, tile_size, rank, world,
                                       ddim_views, true, rgb, alpha, x_prev, packed_rgb, packed_alpha,
                                       packed_x_prev, reinterpret_cast<cudaStream_t>(stream)),
                     "tiles_pack launch");
}

dmv3d_status dmv3d_tiles_unpack(const dmv3d_cameras *cams, int32_t tile_size, int32_t world,
                                int32_t ddim_views, const float *packed_rgb,
                                const float *packed_alpha, const float *packed_x_prev,
                                float *rgb, float *alpha, float *x_prev, dmv3d_stream stream) {
  g_err.clear();
  dmv3d_status s = check_tiles(cams, tile_size, world, ddim_views, packed_rgb, rgb, packed_alpha, alpha,
                               packed_x_prev, x_prev);
  if (s != DMV3D_OK) return s;
  return cuda_status(launch_tiles_copy(cams->num_views, cams->height, cams->width, tile_size, -1, world,
                                       ddim_views, false, packed_rgb, packed_alpha, packed_x_prev, rgb,
                                       alpha, x_prev, reinterpret_cast<cudaStream_t>(stream)),
                     "tiles_unpack launch");
}

dmv3d_status dmv3d_range_flags(const void *workspace, uint32_t *flags, dmv3d_stream stream) {
  g_err.clear();
  CHECK_ARG(workspace && flags, "range_flags: NULL argument");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemcpyAsync(flags, static_cast<const uint32_t *>(workspace) + 1, sizeof(uint32_t),
                                  cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  return cuda_status(e, "range_flags");
}

dmv3d_status dmv3d_workspace_range_flags(dmv3d_workspace *ws, uint32_t *flags) {
  g_err.clear();
  CHECK_ARG(ws && flags, "workspace_range_flags: NULL argument");
  *flags = 0;
  if (!ws->tc_ws) return DMV3D_OK;  // the last step ran on the fp32 SIMT engine
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess)
    e = cudaMemcpy(flags, static_cast<const uint32_t *>(ws->tc_ws) + 1, sizeof(uint32_t), cudaMemcpyDeviceToHost);
  return cuda_status(e, "workspace_range_flags");
}

dmv3d_status dmv3d_select_engine(const dmv3d_triplane *triplane, const dmv3d_mlp *mlp,
                                 const dmv3d_render_opts *opts, int32_t num_assets,
                                 dmv3d_engine *engine) {
  g_err.clear();
  dmv3d_status s;
  CHECK_ARG(engine != nullptr, "select_engine: engine is NULL");
  if ((s = check_triplane(triplane)) != DMV3D_OK) return s;
  CHECK_ARG(opts != nullptr, "opts is NULL");
  if ((s = check_mlp(mlp, triplane, opts->agg)) != DMV3D_OK) return s;
  CHECK_ARG(num_assets >= 1, "select_engine: num_assets must be >= 1");
  Engine e;
  if ((s = pick_engine(triplane, mlp, opts, e, num_assets)) != DMV3D_OK) return s;
  *engine = e == Engine::TC ? DMV3D_ENGINE_TCGEN05 : DMV3D_ENGINE_SIMT;
  return DMV3D_OK;
}

dmv3d_status dmv3d_render_ddim_step_host(dmv3d_workspace *ws, const dmv3d_triplane *triplane,
                                         const dmv3d_cameras *cams, const dmv3d_mlp *mlp,
                                         const dmv3d_render_opts *opts,
                                         const dmv3d_ddim_params *ddim, const float *x_t,
                                         const float *z, float *x_prev, float *rgb, float *alpha,
                                         dmv3d_stream stream) {
  g_err.clear();
  CHECK_ARG(ws != nullptr, "ws is NULL");
  CHECK_ARG(triplane && cams && mlp && opts && ddim, "NULL argument");
  CHECK_ARG(triplane->data && cams->intrinsics && cams->c2w && x_t && x_prev, "NULL host buffer");
  CHECK_ARG(mlp->num_layers >= 2 && mlp->num_layers <= kMaxLayers, "mlp: num_layers must be in [2, 8]");
  CHECK_ARG(mlp->weights && mlp->biases, "mlp: weights / biases array is NULL");
  CHECK_ARG(cams->num_views >= 1 && cams->height >= 1 && cams->width >= 1, "cameras: V, H, W must be >= 1");
  CHECK_ARG(ddim->ddim_views >= 1 && ddim->ddim_views <= cams->num_views, "ddim: need 1 <= ddim_views <= V");
  if (opts->tile_size)  // the full outputs are copied back: a tile shard would return stale pixels
    return fail(DMV3D_ERR_UNSUPPORTED, "host step: interleaved tiles are a device-buffer option");
  {  // validate everything the copies and the launch depend on BEFORE any work is enqueued
    dmv3d_status s0;
    if ((s0 = check_cams(cams)) != DMV3D_OK) return s0;
    if ((s0 = check_triplane(triplane)) != DMV3D_OK) return s0;
    const int64_t nr = (int64_t)cams->num_views * cams->height * cams->width;
    if ((s0 = check_opts(opts, nr)) != DMV3D_OK) return s0;
    if ((s0 = check_mlp(mlp, triplane, opts->agg)) != DMV3D_OK) return s0;
    if (ddim->ddim_views > 64) return fail(DMV3D_ERR_UNSUPPORTED, "ddim: at most 64 DDIM views per call");
    DdimCoef k0;
    if ((s0 = ddim_coefficients(ddim, ddim->ddim_views, k0)) != DMV3D_OK) return s0;
    CHECK_ARG(k0.sigma_t == 0.0f || z != nullptr || ddim->noise_in_kernel,
              "ddim: eta > 0 needs z or noise_in_kernel");
    dmv3d_render_opts oe = *opts;  // the workspace the step will provide if none is given
    if (!oe.workspace) {
      oe.workspace = reinterpret_cast<void *>(uintptr_t(256));
      oe.workspace_bytes = dmv3d_workspace_bytes(triplane, mlp);
      if (!oe.workspace_bytes) oe.workspace = nullptr;
    }
    Engine en;
    if ((s0 = pick_engine(triplane, mlp, &oe, en)) != DMV3D_OK) return s0;
  }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const size_t V = cams->num_views, HW = (size_t)cams->height * cams->width;
  const size_t tp_bytes = (size_t)3 * triplane->res * triplane->res * triplane->channels *
                          (triplane->dtype == DMV3D_F32 ? 4 : triplane->dtype == DMV3D_BF16 ? 2 : 1);
  const size_t img_in = (size_t)ddim->ddim_views * 3 * HW * 4;
  cudaError_t e = cudaSuccess;
#define TRY(x)                                                  \
  do {                                                          \
    e = (x);                                                    \
    if (e != cudaSuccess) return cuda_status(e, "host step");   \
  } while (0)
  TRY(ws_reserve(ws->tp, tp_bytes));
  TRY(ws_reserve(ws->intr, V * 16));
  TRY(ws_reserve(ws->c2w, V * 48));
  TRY(ws_reserve(ws->xt, img_in));
  TRY(ws_reserve(ws->xp, img_in));
  if (z) TRY(ws_reserve(ws->z, img_in));
  if (rgb) TRY(ws_reserve(ws->rgb, V * 3 * HW * 4));
  if (alpha) TRY(ws_reserve(ws->alpha, V * HW * 4));
  TRY(cudaMemcpyAsync(ws->tp.p, triplane->data, tp_bytes, cudaMemcpyHostToDevice, st));
  TRY(cudaMemcpyAsync(ws->intr.p, cams->intrinsics, V * 16, cudaMemcpyHostToDevice, st));
  TRY(cudaMemcpyAsync(ws->c2w.p, cams->c2w, V * 48, cudaMemcpyHostToDevice, st));
  TRY(cudaMemcpyAsync(ws->xt.p, x_t, img_in, cudaMemcpyHostToDevice, st));
  if (z) TRY(cudaMemcpyAsync(ws->z.p, z, img_in, cudaMemcpyHostToDevice, st));
  const void *dw[kMaxLayers];
  const float *db[kMaxLayers];
  const size_t wel = mlp->dtype == DMV3D_BF16 ? 2 : 4;
  for (int l = 0; l < mlp->num_layers; ++l) {
    const size_t in = l == 0 ? mlp->in_dim : mlp->hidden;
    const size_t out = l == mlp->num_layers - 1 ? 4 : mlp->hidden;
    CHECK_ARG(mlp->weights[l] && mlp->biases[l], "mlp: a layer pointer is NULL");
    TRY(ws_reserve(ws->w[l], in * out * wel));
    TRY(ws_reserve(ws->b[l], out * 4));
    TRY(cudaMemcpyAsync(ws->w[l].p, mlp->weights[l], in * out * wel, cudaMemcpyHostToDevice, st));
    TRY(cudaMemcpyAsync(ws->b[l].p, mlp->biases[l], out * 4, cudaMemcpyHostToDevice, st));
    dw[l] = ws->w[l].p;
    db[l] = static_cast<const float *>(ws->b[l].p);
  }
  dmv3d_triplane t = *triplane;
  t.data = ws->tp.p;
  dmv3d_cameras c = *cams;
  c.intrinsics = static_cast<const float *>(ws->intr.p);
  c.c2w = static_cast<const float *>(ws->c2w.p);
  dmv3d_mlp m = *mlp;
  m.weights = dw;
  m.biases = db;
  dmv3d_render_opts o = *opts;
  if (!o.workspace) {
    const uint64_t need = dmv3d_workspace_bytes(&t, &m);
    if (need) {
      TRY(ws_reserve(ws->scratch, need));
      o.workspace = ws->scratch.p;
      o.workspace_bytes = need;
    }
  }
  // Render in view chunks (ray ranges on view boundaries: the same patches, hence the same
  // bits as one launch); each chunk's outputs are copied back on the copy stream while the
  // next chunk renders.  The projected triplane G is computed by the first launch only.
  int cur_dev = 0;
  TRY(cudaGetDevice(&cur_dev));
  if (ws->copy == nullptr || ws->dev != cur_dev) {
    if (ws->copy) {
      cudaStreamDestroy(ws->copy);
      for (auto &ev : ws->ev) cudaEventDestroy(ev);
    }
    TRY(cudaStreamCreateWithFlags(&ws->copy, cudaStreamNonBlocking));
    for (auto &ev : ws->ev) TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    ws->dev = cur_dev;
  }
  const int nc = (int)(V < (size_t)dmv3d_workspace::kChunks ? V : (size_t)dmv3d_workspace::kChunks);
  const size_t vpc = (V + nc - 1) / nc;
  const size_t dv = (size_t)ddim->ddim_views;
  const bool tc = o.workspace != nullptr && o.engine != DMV3D_ENGINE_SIMT;
  ws->tc_ws = tc ? o.workspace : nullptr;
  for (int k = 0; k < nc; ++k) {
    const size_t v0 = k * vpc, v1 = (v0 + vpc < V) ? v0 + vpc : V;
    if (v0 >= v1) break;
    dmv3d_render_opts ok = o;
    ok.ray_begin = (int64_t)(v0 * HW);
    ok.ray_end = (int64_t)(v1 * HW);
    const dmv3d_status s = render_impl(&t, &c, &m, &ok, ddim, static_cast<const float *>(ws->xt.p),
                                       z ? static_cast<const float *>(ws->z.p) : nullptr,
                                       static_cast<float *>(ws->xp.p),
                                       rgb ? static_cast<float *>(ws->rgb.p) : nullptr,
                                       alpha ? static_cast<float *>(ws->alpha.p) : nullptr, st,
                                       tc && k > 0);
    if (s != DMV3D_OK) return s;
    TRY(cudaEventRecord(ws->ev[k], st));
    TRY(cudaStreamWaitEvent(ws->copy, ws->ev[k], 0));
    const size_t x0 = v0 < dv ? v0 : dv, x1 = v1 < dv ? v1 : dv;
    if (x1 > x0)
      TRY(cudaMemcpyAsync(x_prev + x0 * 3 * HW, static_cast<float *>(ws->xp.p) + x0 * 3 * HW,
                          (x1 - x0) * 3 * HW * 4, cudaMemcpyDeviceToHost, ws->copy));
    if (rgb)
      TRY(cudaMemcpyAsync(rgb + v0 * 3 * HW, static_cast<float *>(ws->rgb.p) + v0 * 3 * HW,
                          (v1 - v0) * 3 * HW * 4, cudaMemcpyDeviceToHost, ws->copy));
    if (alpha)
      TRY(cudaMemcpyAsync(alpha + v0 * HW, static_cast<float *>(ws->alpha.p) + v0 * HW,
                          (v1 - v0) * HW * 4, cudaMemcpyDeviceToHost, ws->copy));
  }
  // the caller's stream completes after the last copy
  TRY(cudaEventRecord(ws->ev[dmv3d_workspace::kChunks], ws->copy));
  TRY(cudaStreamWaitEvent(st, ws->ev[dmv3d_workspace::kChunks], 0));
#undef TRY
  return DMV3D_OK;
}

}  // extern "C"
