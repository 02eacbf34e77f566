// kernels.h -- internal launchers of libdmv3d (not part of the C ABI).
#pragma once
#include <cuda_runtime.h>

#include "common.cuh"

namespace dmv3d {

constexpr int kSimtThreads = 128;

// api.cu: CUDA-event bracket around the dominant (render) kernel of a call
void timer_begin(void *timer, cudaStream_t st);
void timer_end(void *timer, cudaStream_t st);

// render_simt.cu
bool simt_supported(int K, int HD, bool concat);
size_t simt_smem_bytes(int K, int HD, int L);
cudaError_t launch_render_simt(const RenderParams &P, bool tp_bf16, bool w_bf16,
                               cudaStream_t st);
cudaError_t launch_features(const RenderParams &P, bool tp_bf16, int64_t n, const float *pts,
                            float *out, cudaStream_t st);
cudaError_t launch_decode(const RenderParams &P, bool tp_bf16, bool w_bf16, int64_t n,
                          const float *pts, float *out, cudaStream_t st);
cudaError_t launch_density_grid(const RenderParams &P, bool tp_bf16, bool w_bf16, int G,
                                float *sigma, float *rgb, cudaStream_t st);

// backward.cu (row f1)
struct GradParams {
  const float *g_rgb;    // [V][3][H][W]
  const float *g_alpha;  // [V][H][W] or null
  float *dF;             // [3][R][R][C], fp32, accumulated
  float *dW[kMaxLayers];  // [out][in], accumulated
  float *db[kMaxLayers];  // [out], accumulated
  const float *fwd_rgb;   // optional forward render (C per ray) ...
  const float *fwd_alpha; // ... and alpha (T_N = 1 - alpha): skips the first march
};
bool backward_supported(int K, int HD, int L, bool concat);
cudaError_t launch_render_backward(const RenderParams &P, const GradParams &Gp, bool tp_bf16,
                                   bool w_bf16, cudaStream_t st);

// render_tc.cu (tcgen05 / TMEM engine).  Workspace: [256-B header: patch counter]
// [G: (3 R R + 1) x HD fp16] (+ for the backward, 256-B aligned: [dG: (3 R R + 1) x HD fp32])
constexpr uint32_t kTcWsHeader = 256;
bool tc_supported(int C, int HD, int L);  // C = triplane channels per plane
size_t tc_workspace_bytes(int R, int HD, int assets = 1);  // render: header + assets x G
cudaError_t launch_preproject(const RenderParams &P, cudaStream_t st);
cudaError_t launch_render_tc(const RenderParams &P, cudaStream_t st);

// backward_tc.cu (row f1 on the tensor cores)
size_t tc_backward_workspace_bytes(int R, int HD);
bool tc_backward_supported(int C, int HD, int L);
cudaError_t launch_render_backward_tc(const RenderParams &P, const GradParams &Gp, cudaStream_t st);

// elementwise.cu
struct DdimCoef {
  float x0_scale, x0_shift, sqrt_ab_t, inv_sqrt_1m_ab_t, sqrt_ab_p, c_eps, sigma_t;
  uint64_t keep_bits;
  uint64_t noise_seed;  // used when z == null and sigma_t != 0 (in-kernel noise, row f4)
};
cudaError_t launch_ddim(const DdimCoef &c, int V, int H, int W, const float *x_t,
                        const float *x0_rgb, const float *z, const uint8_t *keep_dev,
                        float *x_prev, cudaStream_t st);
cudaError_t launch_plucker(const RenderParams &P, float *out, cudaStream_t st);
// interleaved-tile merge: pack (rank's tiles, image -> blocks) or unpack (every rank's
// gathered blocks -> images); src / dst are (rgb, alpha, x_prev) triples
cudaError_t launch_tiles_copy(int V, int H, int W, int T, int rank, int world, int ddim_views, bool pack,
                              const float *src_rgb, const float *src_alpha, const float *src_xp,
                              float *dst_rgb, float *dst_alpha, float *dst_xp, cudaStream_t st);
cudaError_t launch_ray_geometry(const RenderParams &P, float *o_d, float *tn_tf, uint8_t *hit,
                                cudaStream_t st);
cudaError_t launch_sample_points(const RenderParams &P, float *t_k, float *points,
                                 int32_t *texel, float *frac, cudaStream_t st);

}  // namespace dmv3d
