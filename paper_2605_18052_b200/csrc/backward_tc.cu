// backward_tc.cu -- the renderer backward on the tcgen05 tensor
// cores: gradients of L = <g_rgb, rgb> + <g_alpha, alpha> w.r.t. the triplane and
// the shared MLP (the "differentiable volume rendering" L_recon trains through,
// PAPER.md:47-55, :71), through the same rays, samples, projected-triplane blend and
// fp16 MLP MMAs as the forward tensor-core engine (render_tc.cu).
//
// The first layer is folded into the triplane as in the forward, G = F W0^T + b0 (K0,
// per texel), z0_s = sum_t a_{s,t} G_t with the sparse bilinear weights a.  So the
// gradient is accumulated in the 64-wide projected space and mapped back after the
// render kernel:
//     dG_t = sum_s a_{s,t} dz0_s,   dF_t = W0^T dG_t,   dW0 = sum_t dG_t F_t^T,
//     db0 = bscale sum_t dG_t (+ the half-pixel mode's bias row).
//
// K1 `render_bwd_tc_kernel`: persistent, one CTA per SM, NG groups of 4 warps, a
// group owns a 4x4-pixel patch (16 rays) and walks it twice in chunks of 8 samples
// (tile = 128 rows = 16 rays x 8 samples):
//   pass 1: forward (blend MMA + L-1 layer MMAs) and compositing -> C = sum w c + T_N bg
//           and T_N per ray (skipped when the caller passes its forward's rgb / alpha);
//   pass 2: forward again, keeping every layer's fp16 input h_l in shared memory,
//           then per sample dC/dtau_k = T_{k+1} c_k - R_k, R_k = C - sum_{j<=k} w_j c_j
//           (8-lane scans), dC/dc_k = w_k, dA/dtau_k = T_N -> the head delta d_o
//           (fp16 tile), and back through the MLP as MMAs, M = 128 samples:
//             dh_l  = dz_l W_l                       (A = dz_l K-major, B = W_l MN-major)
//             dW_l^T, db_l += [h_l | 1]^T dz_l       (A = h_l tile MN-major: the same
//                                                     bytes the forward reads K-major)
//             dz_{l-1} = dh_l (.) [h_l > 0]          (written over h_l's tile)
//             dG_window = A_blend^T dz0              (the blend's own sparse A tile,
//                                                     MN-major; rows = staged texels)
//           dG rows go to the workspace with 16-B vector reductions; each group's dW/db
//           accumulators live in TMEM for the whole launch and are added to the
//           caller's buffers once per CTA.  The dh and dW K-steps of a trip are issued
//           interleaved (independent accumulation chains overlap in the tensor pipe;
//           one chain's dependent steps do not).
// K2/K3 map dG back to dF, dW0 and db0 (fp32 CUDA cores, 2 x 63 MFLOP at R = 64).
//
// Shared-memory operand layouts are SWIZZLE_NONE core matrices (8 rows x 16 B):
// for either major-ness LBO = stride between core matrices along K and SBO = along
// M/N (tools/mma_layout_check.cu verifies this on the B200).  A tile written by its
// row threads as [row][col] with 16-B chunks of 8 columns serves both as a K-major
// operand (rows = M) and as an MN-major one (rows = K).
// opts.term_eps > 0 differentiates the early-terminated render (the forward's rule, per
// 8-sample chunk); otherwise the full quadrature.  Exact up to the fp16 operand rounding
// (tolerances).
#include <cuda_fp16.h>
#include <cuda_fp8.h>

#include "common.cuh"
#include "kernels.h"
#include "tc_ptx.cuh"

namespace dmv3d {

namespace {

constexpr int kHD = 64;        // hidden width
constexpr int kKW = 96;        // max staged texels per blend window (128^2 crops: most chunks fit)
constexpr int kPatch = 4;      // 4x4 rays per patch
constexpr int kChunk = 8;      // samples per ray per tile
constexpr uint32_t kHK = kHD + 16;          // h tile columns: 64 activations + [1, 0 x 15]
constexpr uint32_t kHSbo = (kHK / 8) * 128;   // 1280: stride of 8-row groups in an h tile
constexpr uint32_t kHBytes = 128 * kHK * 2;   // 20 KiB
// sparse A tile: 8-row groups (kKW / 8) * 128 + 32 B apart, so rows m, m+8, m+16, m+24 of
// a warp fall into different banks in the 2-byte weight scatter (as in render_tc); the
// tile is rounded up to whole KiB so every group's B tile stays 1 KiB aligned
constexpr uint32_t kASbo = (kKW / 8) * 128 + 32;                // 1568
constexpr uint32_t kABytes = ((16 * kASbo + 1023) / 1024) * 1024;  // 25 KiB
constexpr uint32_t kBBytes = kKW * kHD * 2;   // 12 KiB (SWIZZLE_128B texel rows); later d_o
constexpr uint32_t kDoSbo = 256;              // d_o tile [128][16]: 2 column blocks
constexpr uint32_t kWK = kHD + 16;
constexpr uint32_t kWSbo = (kWK / 8) * 128;   // 1280
constexpr uint32_t kWHidden = kHD * kWK * 2;  // 10 KiB
constexpr uint32_t kWHead = 16 * kWK * 2;     // 2.5 KiB
constexpr size_t kSmemLimit = 232448;

template <int NG>
struct BwShared {
  uint64_t mbar[NG];
  uint64_t mbar2[NG];  // the weight-gradient chain, issued by a second thread of the group
  uint32_t tmem_base;
  int patch[NG];
  int bbox[NG][2][8];
  int coltex[NG][kKW];
  float head_bias[4];
};

__host__ __device__ constexpr uint32_t group_bytes(int L) {
  return kBBytes + kABytes + (uint32_t)(L - 1) * kHBytes;
}
template <int NG>
size_t bw_smem_bytes(int L) {
  return 1024 + (size_t)NG * group_bytes(L) + (size_t)(L - 2) * kWHidden + kWHead +
         sizeof(BwShared<NG>);
}

__host__ __device__ constexpr uint32_t idesc(uint32_t M, uint32_t N, uint32_t a_mn, uint32_t b_mn) {
  return ptx::idesc_f16(M, N, b_mn) | (a_mn << 15);
}

__device__ __forceinline__ void red_add_v4(float *p, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c),
               "f"(d)
               : "memory");
}
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(addr)
               : "memory");
  return v;
}
// dz = dh where h > 0 (fp16 h, fp32 dh), packed fp16: one cvt, one HSET2, one LOP
__device__ __forceinline__ uint32_t mask_pack(uint32_t h2, float d0, float d1) {
  const __half2 h = *reinterpret_cast<const __half2 *>(&h2);
  return ptx::pack_f16x2(d0, d1) & __hgt2_mask(h, __float2half2_rn(0.0f));
}

// the forward tensor-core engine's head activations (fast exp / divide)
__device__ __forceinline__ float softplus_fast(float x) {
  return __logf(1.0f + __expf(-fabsf(x))) + fmaxf(x, 0.0f);
}
__device__ __forceinline__ float sigmoid_fast(float x) { return __fdividef(1.0f, 1.0f + __expf(-x)); }

}  // namespace

size_t tc_backward_workspace_bytes(int R, int HD) {
  const size_t g = (tc_workspace_bytes(R, HD) + 255) & ~size_t(255);
  return g + ((size_t)3 * R * R + 1) * HD * 4;
}

bool tc_backward_supported(int C, int HD, int L) {
  return tc_supported(C, HD, L) && bw_smem_bytes<1>(L) <= kSmemLimit &&
         kHD + (L - 2) * kHD + 16 + 48 <= 512;
}

template <int NG>
__global__ void __launch_bounds__(128 * NG, 1)
    render_bwd_tc_kernel(const __grid_constant__ RenderParams P,
                         const __grid_constant__ GradParams Gp, float *__restrict__ dG) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~uintptr_t(1023));
  const int L = P.L;
  const int tid_cta = threadIdx.x;
  const int warp = __shfl_sync(0xffffffffu, tid_cta >> 5, 0);  // warp-uniform (see render_tc)
  const int g = warp >> 2;
  const int tid = tid_cta & 127;
  const int bar_id = 1 + g;
  uint8_t *gbase = smem + (size_t)g * group_bytes(L);
  uint8_t *wsm = smem + (size_t)NG * group_bytes(L);
  __shared__ BwShared<NG> sh_s;  // static: LDS/STS/ATOMS rather than generic accesses
  BwShared<NG> *sh = &sh_s;

  const uint32_t sB = ptx::smem_u32(gbase);             // staged texels, then d_o
  const uint32_t sA = sB + kBBytes;                      // sparse blend A
  const uint32_t sH = sA + kABytes;                      // h_1 .. h_{L-1} (then dz)
  const uint32_t sW = ptx::smem_u32(wsm);
  auto hT = [&](int l) { return sH + (uint32_t)(l - 1) * kHBytes; };  // tile of h_l, l >= 1

  // ---- prologue: barriers, TMEM, weights, the constant [1, 0...] columns of the h tiles
  if (tid_cta == 0) {
    for (int i = 0; i < NG; ++i) {
      ptx::mbar_init(&sh->mbar[i], 1);
      ptx::mbar_init(&sh->mbar2[i], 1);
    }
    for (int i = 0; i < NG; ++i)
      for (int p = 0; p < 2; ++p)
        for (int e = 0; e < 8; ++e) sh->bbox[i][p][e] = (e < 4) ? 0x7fffffff : -1;
    ptx::fence_mbar_init();
  }
  const uint32_t ndw = (uint32_t)(L - 2) * kHD + 16;  // dW^T accumulators: 64 cols per hidden layer, 16 for the head
  if (warp == 0) ptx::tmem_alloc(&sh->tmem_base, 512);
  for (int l = 1; l < L; ++l) {
    const int nout = (l == L - 1) ? 16 : kHD;
    const int nreal = (l == L - 1) ? 4 : kHD;
    uint8_t *wl = wsm + (l - 1) * kWHidden;
    const __nv_bfloat16 *W = reinterpret_cast<const __nv_bfloat16 *>(P.w[l]);
    for (int e = tid_cta; e < nout * (int)kWK; e += 128 * NG) {
      const int n = e / kWK, k = e - n * kWK;
      float v = 0.0f;
      if (n < nreal) {
        if (k < kHD) v = __bfloat162float(W[n * kHD + k]);
        else if (k == kHD) v = __ldg(P.b[l] + n);
      }
      const uint32_t off = (n >> 3) * kWSbo + (k >> 3) * 128 + (n & 7) * 16 + (k & 7) * 2;
      *reinterpret_cast<__half *>(wl + off) = __float2half_rn(v);
    }
  }
  if (tid_cta < 4) sh->head_bias[tid_cta] = __ldg(P.b[L - 1] + tid_cta);
  {
    const uint32_t rowoff = (uint32_t)((tid >> 3) * kHSbo + (tid & 7) * 16);
    for (int l = 1; l < L; ++l) {
      ptx::sts128(hT(l) + rowoff + 8 * 128, 0x3C00u, 0u, 0u, 0u);  // column 64 = 1.0
      ptx::sts128(hT(l) + rowoff + 9 * 128, 0u, 0u, 0u, 0u);
    }
  }
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  // TMEM per group: the accumulator (z / dh / dG) and the group's own dW^T accumulators
  // (not shared between groups: accumulating into one region would chain the groups' MMAs)
  // + 48 columns: the forward pass's fp16 activation operand (32 columns of h_l, the
  // constant bias K block, padding) -- the forward MMAs read A from TMEM, so the h tiles
  // written for the backward's MMAs need no proxy fence until the first backward trip
  const uint32_t gcols = kHD + ndw + 48u;
  const uint32_t tmem = sh->tmem_base + (uint32_t)g * gcols;
  const uint32_t tmem_dw = tmem + (uint32_t)kHD;
  const uint32_t tmem_a = tmem + kHD + ndw;  // activation operand (lane = row)
  const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
  const uint32_t tmem_row = tmem + lane_off;
  {  // zero this group's dW accumulators (its 4 warps cover the 128 lanes)
    const uint32_t z[16] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
    for (uint32_t c = 0; c < ndw; c += 16) ptx::tmem_st16(tmem_dw + lane_off + c, z);
    const uint32_t bias[8] = {0x3C00u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};  // k = 64: 1.0
    ptx::tmem_st8(tmem_a + lane_off + kHD / 2, bias);
    ptx::tmem_st_wait();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();

  constexpr uint32_t id_blend = idesc(128, kHD, 0, 1);
  constexpr uint32_t id_hidden = idesc(128, kHD, 0, 0);
  constexpr uint32_t id_head = idesc(128, 16, 0, 0);
  constexpr uint32_t id_dh = idesc(128, kHD, 0, 1);     // A = dz (K-major), B = W (MN-major)
  constexpr uint32_t id_dw = idesc(128, kHD, 1, 1);     // A = h^T, B = dz (both MN-major)
  constexpr uint32_t id_dw_head = idesc(128, 16, 1, 1);
  constexpr uint32_t id_dg = idesc(128, kHD, 1, 1);     // A = A_blend^T, B = dz0

  const __half *G = reinterpret_cast<const __half *>(reinterpret_cast<const uint8_t *>(P.ws) +
                                                      kTcWsHeader);
  unsigned int *counter = reinterpret_cast<unsigned int *>(P.ws);

  const int64_t HW = (int64_t)P.H * P.W;
  const int v_lo = (int)(P.ray_begin / HW);
  const int v_hi = (int)((P.ray_end - 1) / HW);
  const int PH = (P.H + kPatch - 1) / kPatch, PW = (P.W + kPatch - 1) / kPatch;
  const int64_t npatch = (int64_t)(v_hi - v_lo + 1) * PH * PW;
  const int slot = tid >> 3, q = tid & 7;
  const int R = P.R;
  const float wscale = (P.agg == 0) ? (1.0f / 3.0f) : 1.0f;
  const int hb = P.smode != 0 ? 1 : 0;
  const bool fastgeo = P.smode == 0 && P.inv_ext[0] != 0.0f && P.inv_ext[1] != 0.0f && P.inv_ext[2] != 0.0f;
  const float rm1 = __int2float_rn(R - 1);
  const uint32_t sArow = sA + (uint32_t)((tid >> 3) * kASbo + (tid & 7) * 16);
  const uint32_t hrow = (uint32_t)((tid >> 3) * kHSbo + (tid & 7) * 16);
  const uint32_t dorow = sB + (uint32_t)((tid >> 3) * kDoSbo + (tid & 7) * 16);
  uint32_t mphase = 0;
  int chunk_ctr = 0;

  auto mma_wait = [&]() {
    ptx::mbar_wait(&sh->mbar[g], mphase);
    mphase ^= 1u;
    ptx::tc_fence_after();
  };
  // backward trips: the dh chain (thread 0, mbar) and the dW chain (thread 32, mbar2) are
  // issued by two threads, so their instruction issue overlaps
  uint32_t mphase2 = 0;
  auto mma_wait2 = [&]() {
    ptx::mbar_wait(&sh->mbar[g], mphase);
    mphase ^= 1u;
    ptx::mbar_wait(&sh->mbar2[g], mphase2);
    mphase2 ^= 1u;
    ptx::tc_fence_after();
  };
  // all rows' smem / TMEM accesses done -> the elected thread may issue
  auto sync_for_mma = [&]() {
    ptx::fence_proxy_async_smem();
    ptx::tc_fence_before();
    ptx::bar_sync(bar_id, 128);
  };

  while (true) {
    if (tid == 0) sh->patch[g] = (int)atomicAdd(counter, 1u);
    ptx::bar_sync(bar_id, 128);
    const int64_t patch = sh->patch[g];
    if (patch >= npatch) break;
    const int v = v_lo + (int)(patch / ((int64_t)PH * PW));
    const int prem = (int)(patch % ((int64_t)PH * PW));
    const int i = (prem / PW) * kPatch + (slot >> 2);
    const int j = (prem % PW) * kPatch + (slot & 3);
    const int64_t r = (int64_t)v * HW + (int64_t)i * P.W + j;
    const bool pix = (i < P.H) && (j < P.W) && r >= P.ray_begin && r < P.ray_end;
    Ray ray;
    ray.hit = false;
    ray.t_near = ray.t_far = 0.0f;
    if (pix) ray = make_ray(P.intr, P.c2w, v, i, j, P.lo, P.hi);
    bool alive = pix && ray.hit;  // cleared when the ray terminates (T < term_eps)
    if (!ptx::bar_red_or(bar_id, 128, alive)) continue;
    const float delta = alive ? sample_delta(ray, P.N) : 0.0f;
    float gr[3] = {0.f, 0.f, 0.f}, gA = 0.0f;
    if (alive) {
      const int64_t px = (int64_t)i * P.W + j;
#pragma unroll
      for (int c = 0; c < 3; ++c) gr[c] = __ldg(Gp.g_rgb + ((int64_t)v * 3 + c) * HW + px);
      if (Gp.g_alpha) gA = __ldg(Gp.g_alpha + (int64_t)v * HW + px);
    }

    // per-chunk state of this row's sample (set by geometry())
    bool sv = false;
    int ix[3];
    float wl[3], wh[3];
    int lo0, lo1, lo2, ext0, ext1, ext2, ktex, ktot;

    // sample point, texel cells, group bounding box of the chunk at k0
    auto geometry = [&](int k0) {
      const int par = chunk_ctr & 1;
      ++chunk_ctr;
      const int k = k0 + q;
      sv = alive && k < P.N;
      ix[0] = ix[1] = ix[2] = 0;
      wl[0] = wl[1] = wl[2] = 0.f;
      wh[0] = wh[1] = wh[2] = 0.f;
      if (sv) {
        float p[3];
        const float u = P.jitter ? jitter_u(P.seed, (uint64_t)r * P.N + k) : 0.5f;
        sample_p(ray, sample_t(ray, delta, k, u), p);
        if (fastgeo) {  // align-corners, power-of-two extents: texel_coord's multiply path
                        // inline, no per-axis branches (same IEEE ops; see render_tc)
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            const float sx = __fmul_rn(__fsub_rn(p[a], P.lo[a]), P.inv_ext[a]);
            const float px = fminf(fmaxf(__fmul_rn(sx, rm1), 0.0f), rm1);
            const int i0 = min(__float2int_rd(px), R - 2);
            const float f = __fsub_rn(px, __int2float_rn(i0));
            ix[a] = i0;
            wl[a] = 1.0f - f;
            wh[a] = f;
          }
        } else {
#pragma unroll
          for (int a = 0; a < 3; ++a)
            texel_axis(p[a], P.lo[a], P.hi[a], P.inv_ext[a], R, P.smode, ix[a], wl[a], wh[a]);
        }
      }
      int mn[3], mx[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        mn[a] = __reduce_min_sync(0xffffffffu, sv ? ix[a] : 0x7fffffff);
        mx[a] = __reduce_max_sync(0xffffffffu, sv ? ix[a] : -1);
      }
      if ((tid & 31) == 0) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          atomicMin(&sh->bbox[g][par][a], mn[a]);
          atomicMax(&sh->bbox[g][par][4 + a], mx[a]);
        }
      }
      ptx::bar_sync(bar_id, 128);
      const int *bb = sh->bbox[g][par];
      lo0 = bb[0];
      lo1 = bb[1];
      lo2 = bb[2];
      ext0 = bb[4] - lo0 + 2;
      ext1 = bb[5] - lo1 + 2;
      ext2 = bb[6] - lo2 + 2;
      ktex = ext0 * ext1 + ext0 * ext2 + ext1 * ext2;
      ktot = ktex + hb;
      if (tid < 8) sh->bbox[g][par ^ 1][tid] = (tid < 4) ? 0x7fffffff : -1;
      if (ktot <= 0 || ktot > (1 << 20)) ktot = 0;  // no alive sample: empty box
    };

    // column -> texel table of window [w0, w0 + kpad); optionally stage the texel rows
    // of G into the B tile (SWIZZLE_128B MN-major)
    auto fill_table = [&](int w0, bool stage) {
      const int base1 = ext0 * ext1, base2 = base1 + ext0 * ext2;
      const int kpad = (min(kKW, ktot - w0) + 15) & ~15;
      if (tid < kpad) {
        const int kg = w0 + tid;
        int texel = -1;
        if (kg == ktex && hb) {
          texel = 3 * R * R;
        } else if (kg < ktex) {
          int loc, bw, ta0, tb0, pl;
          if (kg >= base2) { pl = 2; loc = kg - base2; bw = ext1; ta0 = lo1; tb0 = lo2; }
          else if (kg >= base1) { pl = 1; loc = kg - base1; bw = ext0; ta0 = lo0; tb0 = lo2; }
          else { pl = 0; loc = kg; bw = ext0; ta0 = lo0; tb0 = lo1; }
          // row = floor(loc / bw): loc < 2^13 and bw < 2^8, so an approximate reciprocal
          // is never off by one
          const int rr = (int)(((float)loc + 0.5f) * __fdividef(1.0f, (float)bw));
          texel = (pl * R + tb0 + rr) * R + ta0 + (loc - rr * bw);
        }
        sh->coltex[g][tid] = texel;
        if (stage) {
          const uint32_t drow = sB + (uint32_t)(tid << 7);
          const __half *src = G + (size_t)max(texel, 0) * kHD;
          const uint32_t nb = texel >= 0 ? 16u : 0u;
#pragma unroll
          for (int ch = 0; ch < 8; ++ch)
            ptx::cp_async16(drow + (uint32_t)((ch ^ (tid & 7)) << 4), src + ch * 8, nb);
        }
      }
    };

    // this row's sparse A row of window [w0, w0 + kp): 12 bilinear weights (+ bias column)
    auto scatter_a = [&](int w0) {
      const int kp = min(kKW, ktot - w0);
      const bool one_window = ktot <= kKW;
      // zero the window's kpad columns (a plain loop of two 16-B stores, as in render_tc)
      const int kpz = (kp + 15) & ~15;
#pragma unroll 1
      for (int kc = 0; kc < kpz / 16; ++kc) {
        ptx::sts128(sArow + (uint32_t)(kc << 8), 0u, 0u, 0u, 0u);
        ptx::sts128(sArow + (uint32_t)((kc << 8) + 128), 0u, 0u, 0u, 0u);
      }
      if (!sv) return;
      const int base1 = ext0 * ext1, base2 = base1 + ext0 * ext2;
      const int ca = ix[0] - lo0, cb = ix[1] - lo1, cc = ix[2] - lo2;
      const int cols[3] = {cb * ext0 + ca, base1 + cc * ext0 + ca, base2 + cc * ext1 + cb};
      const int bws[3] = {ext0, ext0, ext1};
      const float la[3] = {wl[0], wl[0], wl[1]}, ha[3] = {wh[0], wh[0], wh[1]};
      const float lb[3] = {wl[1], wl[2], wl[2]}, hb3[3] = {wh[1], wh[2], wh[2]};
#pragma unroll
      for (int pl = 0; pl < 3; ++pl) {
        const float gy = lb[pl] * wscale, fy = hb3[pl] * wscale;
        const int c0 = cols[pl] - w0, c2 = c0 + bws[pl];
        const float w4[4] = {la[pl] * gy, ha[pl] * gy, la[pl] * fy, ha[pl] * fy};
        const int cs[4] = {c0, c0 + 1, c2, c2 + 1};
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (one_window || (unsigned)cs[e] < (unsigned)kp)  // one window holds every column
            ptx::sts16(sArow + (uint32_t)(2 * cs[e] + 112 * (cs[e] >> 3)),  // (c>>3)*128 + (c&7)*2
                       ptx::f32_to_f16(w4[e]));
      }
      if (hb && (unsigned)(ktex - w0) < (unsigned)kp)
        ptx::sts16(sArow + (uint32_t)(2 * (ktex - w0) + 112 * ((ktex - w0) >> 3)),
                   (uint16_t)0x3c00u);
    };

    // forward of the chunk at k0: blend (all windows) + every layer; h_l tiles are left
    // in shared memory.  Returns the head outputs (bias added).
    auto forward = [&](int k0, float o[4]) {
      geometry(k0);
      for (int w0 = 0; w0 < ktot; w0 += kKW) {
        const int kpad = (min(kKW, ktot - w0) + 15) & ~15;
        if (w0 > 0) ptx::bar_sync(bar_id, 128);  // the previous window's table readers are done
        fill_table(w0, true);
        scatter_a(w0);
        ptx::cp_async_wait_all();
        sync_for_mma();
        if (tid < 32) {  // warp 0 issues (elected lane)
          ptx::tc_fence_after();
          for (int ks = 0; ks < kpad / 16; ++ks) {
            const uint64_t ad = ptx::smem_desc(sA + ks * 256, 128, kASbo, 0);
            const uint64_t bd = ptx::smem_desc(sB + ks * 2048, 1024, 1024, 2);
            ptx::mma_f16_ss_warp(tmem, ad, bd, id_blend, (w0 > 0 || ks > 0) ? 1u : 0u);
          }
          ptx::mma_commit_warp(&sh->mbar[g]);
        }
        mma_wait();
      }
      if (ktot == 0) {  // (cannot happen for a patch with an alive sample; keep TMEM defined)
        o[0] = o[1] = o[2] = o[3] = 0.0f;
        return;
      }
      for (int l = 1; l < L; ++l) {
        // z_{l-1} (TMEM) -> h_l = relu(z_{l-1}) fp16 -> this row of h_l's tile
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          uint32_t vv[32];
          ptx::tmem_ld32(tmem_row + 32 * hh, vv);
          ptx::tmem_ld_wait();
          const float *f = reinterpret_cast<const float *>(vv);
          uint32_t pk[16];
#pragma unroll
          for (int c = 0; c < 16; ++c) pk[c] = ptx::pack_relu_f16x2(f[2 * c], f[2 * c + 1]);
#pragma unroll
          for (int c = 0; c < 4; ++c)  // the backward's copy (h_l's smem tile)
            ptx::sts128(hT(l) + hrow + (uint32_t)((4 * hh + c) * 128), pk[4 * c], pk[4 * c + 1],
                        pk[4 * c + 2], pk[4 * c + 3]);
          ptx::tmem_st16(tmem_a + lane_off + 16 * hh, pk);  // the forward MMA's A operand
        }
        ptx::tmem_st_wait();
        ptx::tc_fence_before();
        ptx::bar_sync(bar_id, 128);
        if (tid < 32) {  // warp 0 issues (elected lane)
          ptx::tc_fence_after();
          const uint32_t wbase = sW + (uint32_t)((l - 1) * kWHidden);
          const bool head = l == L - 1;
          const int nks = head ? kHD / 16 : (int)kWK / 16;  // the head's bias is added at readout
          for (int ks = 0; ks < nks; ++ks) {
            const uint64_t bd = ptx::smem_desc(wbase + ks * 256, 128, kWSbo, 0);
            ptx::mma_f16_ts_warp(tmem, tmem_a + ks * 8, bd, head ? id_head : id_hidden, ks > 0 ? 1u : 0u);
          }
          ptx::mma_commit_warp(&sh->mbar[g]);
        }
        mma_wait();
      }
      uint32_t o4[4];
      ptx::tmem_ld4(tmem_row, o4);
      ptx::tmem_ld_wait();
#pragma unroll
      for (int c = 0; c < 4; ++c) o[c] = __uint_as_float(o4[c]) + sh->head_bias[c];
    };

    // ---------------- pass 1: C and T_N of every ray (or the caller's forward render)
    float T = 1.0f, acc[3] = {0.f, 0.f, 0.f};
    const bool have_fwd = Gp.fwd_rgb != nullptr;
    if (have_fwd && alive) {
      const int64_t px = (int64_t)i * P.W + j;
#pragma unroll
      for (int e = 0; e < 3; ++e)  // C = acc + T bg below, with acc := C - bg T_N
        acc[e] = __ldg(Gp.fwd_rgb + ((int64_t)v * 3 + e) * HW + px);
      T = 1.0f - __ldg(Gp.fwd_alpha + (int64_t)v * HW + px);
#pragma unroll
      for (int e = 0; e < 3; ++e) acc[e] = q == 0 ? acc[e] - T * P.bg[e] : 0.0f;
    }
    for (int k0 = 0; k0 < (have_fwd ? 0 : P.N); k0 += kChunk) {
      float o[4];
      forward(k0, o);
      float sigma = 0.0f, c[3] = {0.f, 0.f, 0.f};
      if (sv) {
        sigma = softplus_fast(o[0] + P.dshift);
#pragma unroll
        for (int e = 0; e < 3; ++e) c[e] = sigmoid_fast(o[1 + e]) * (1.0f + 2.0f * P.weps) - P.weps;
      }
      const float tau = sv ? sigma * delta : 0.0f;
      float S = tau;
#pragma unroll
      for (int s = 1; s < kChunk; s <<= 1) {
        const float y = __shfl_up_sync(0xffffffffu, S, s, kChunk);
        if (q >= s) S += y;
      }
      const float w = T * __expf(-(S - tau)) * (-expm1f(-tau));
#pragma unroll
      for (int e = 0; e < 3; ++e) acc[e] += w * c[e];
      T *= __expf(-__shfl_sync(0xffffffffu, S, kChunk - 1, kChunk));
      // early termination, the forward engine's rule: the ray stops after the chunk
      if (alive && P.term_eps > 0.0f && T < P.term_eps) alive = false;
      if (!ptx::bar_red_or(bar_id, 128, alive)) break;
    }
    float Ctot[3];
#pragma unroll
    for (int e = 0; e < 3; ++e) {
#pragma unroll
      for (int s = kChunk / 2; s > 0; s >>= 1) acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], s, kChunk);
      Ctot[e] = acc[e] + T * P.bg[e];
    }
    const float TN = T;

    // ---------------- pass 2: forward again, then back through compositing and the MLP
    T = 1.0f;
    alive = pix && ray.hit;
    float Pc[3] = {0.f, 0.f, 0.f};
    for (int k0 = 0; k0 < P.N; k0 += kChunk) {
      float o[4];
      forward(k0, o);
      // ---- compositing backward (fp32)
      float sigma = 0.0f, zs = 0.0f, c[3] = {0.f, 0.f, 0.f}, sg[3] = {0.f, 0.f, 0.f};
      if (sv) {
        zs = o[0] + P.dshift;
        sigma = softplus_fast(zs);
#pragma unroll
        for (int e = 0; e < 3; ++e) {
          sg[e] = sigmoid_fast(o[1 + e]);
          c[e] = sg[e] * (1.0f + 2.0f * P.weps) - P.weps;
        }
      }
      const float tau = sv ? sigma * delta : 0.0f;
      float S = tau;
#pragma unroll
      for (int s = 1; s < kChunk; s <<= 1) {
        const float y = __shfl_up_sync(0xffffffffu, S, s, kChunk);
        if (q >= s) S += y;
      }
      const float Tk = T * __expf(-(S - tau));
      const float w = Tk * (-expm1f(-tau));
      const float Tk1 = Tk * __expf(-tau);
      float dtau = gA * TN;
#pragma unroll
      for (int e = 0; e < 3; ++e) {
        float sc = w * c[e];
#pragma unroll
        for (int s = 1; s < kChunk; s <<= 1) {
          const float y = __shfl_up_sync(0xffffffffu, sc, s, kChunk);
          if (q >= s) sc += y;
        }
        dtau += gr[e] * (Tk1 * c[e] - (Ctot[e] - (Pc[e] + sc)));
        Pc[e] += __shfl_sync(0xffffffffu, sc, kChunk - 1, kChunk);
      }
      T *= __expf(-__shfl_sync(0xffffffffu, S, kChunk - 1, kChunk));
      const bool stop_after = alive && P.term_eps > 0.0f && T < P.term_eps;
      float d4[4] = {0.f, 0.f, 0.f, 0.f};
      if (sv) {
        const float cs = w * (1.0f + 2.0f * P.weps);
        d4[0] = dtau * delta * sigmoid_fast(zs);
#pragma unroll
        for (int e = 0; e < 3; ++e) d4[1 + e] = gr[e] * cs * sg[e] * (1.0f - sg[e]);
      }
      // d_o row: columns 0..3, zeros to 15 (the B tile is free: the blend completed)
      ptx::sts128(dorow, ptx::pack_f16x2(d4[0], d4[1]), ptx::pack_f16x2(d4[2], d4[3]), 0u, 0u);
      ptx::sts128(dorow + 128, 0u, 0u, 0u, 0u);
      sync_for_mma();
      // ---- head: dh_{L-1} = d_o W_{L-1}; [h_{L-1} | 1]^T d_o -> dW_{L-1}^T, db_{L-1}
      if (tid < 32) {  // warp 0 issues (elected lane)
        ptx::tc_fence_after();
        const uint32_t whead = sW + (uint32_t)((L - 2) * kWHidden);
        ptx::mma_f16_ss_warp(tmem, ptx::smem_desc(sB, 128, kDoSbo, 0), ptx::smem_desc(whead, kWSbo, 128, 0),
                        id_dh, 0u);
        ptx::mma_commit_warp(&sh->mbar[g]);
      } else if (tid < 64) {  // warp 1 issues the dW chain
        ptx::tc_fence_after();
        const uint32_t dcol = tmem_dw + (uint32_t)((L - 2) * kHD);
        for (int ks = 0; ks < 8; ++ks)
          ptx::mma_f16_ss_warp(dcol, ptx::smem_desc(hT(L - 1) + ks * 2 * kHSbo, kHSbo, 128, 0),
                          ptx::smem_desc(sB + ks * 2 * kDoSbo, kDoSbo, 128, 0), id_dw_head, 1u);
        ptx::mma_commit_warp(&sh->mbar2[g]);
      }
      mma_wait2();
      // ---- hidden layers l = L-2 .. 0: dz_l = dh_{l+1} (.) [h_{l+1} > 0] over h_{l+1}'s tile
      for (int l = L - 2; l >= 0; --l) {
        const uint32_t ht = hT(l + 1);
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          uint32_t vv[32];
          ptx::tmem_ld32(tmem_row + 32 * hh, vv);
          ptx::tmem_ld_wait();
          const float *f = reinterpret_cast<const float *>(vv);
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const uint32_t a = ht + hrow + (uint32_t)((4 * hh + c) * 128);
            const uint4 h4 = lds128(a);
            ptx::sts128(a, mask_pack(h4.x, f[8 * c], f[8 * c + 1]), mask_pack(h4.y, f[8 * c + 2], f[8 * c + 3]),
                        mask_pack(h4.z, f[8 * c + 4], f[8 * c + 5]), mask_pack(h4.w, f[8 * c + 6], f[8 * c + 7]));
          }
        }
        sync_for_mma();
        if (l == 0) break;
        // dh_l = dz_l W_l: A = dz_l (K-major, K = 64 outputs), B = W_l as [out][in] MN-major
        // (thread 0); [h_l | 1]^T dz_l -> dW_l^T (rows 0..63), db_l (row 64), K = the 128
        // samples (thread 32): two issuing threads, two mbarriers
        if (tid < 32) {  // warp 0 issues (elected lane)
          ptx::tc_fence_after();
          const uint32_t wbase = sW + (uint32_t)((l - 1) * kWHidden);
          for (int ks = 0; ks < kHD / 16; ++ks)
            ptx::mma_f16_ss_warp(tmem, ptx::smem_desc(ht + ks * 256, 128, kHSbo, 0),
                            ptx::smem_desc(wbase + ks * 2 * kWSbo, kWSbo, 128, 0), id_dh, ks > 0 ? 1u : 0u);
          ptx::mma_commit_warp(&sh->mbar[g]);
        } else if (tid < 64) {  // warp 1 issues the dW chain
          ptx::tc_fence_after();
          const uint32_t dcol = tmem_dw + (uint32_t)((l - 1) * kHD);
          for (int ks = 0; ks < 8; ++ks)
            ptx::mma_f16_ss_warp(dcol, ptx::smem_desc(hT(l) + ks * 2 * kHSbo, kHSbo, 128, 0),
                            ptx::smem_desc(ht + ks * 2 * kHSbo, kHSbo, 128, 0), id_dw, 1u);
          ptx::mma_commit_warp(&sh->mbar2[g]);
        }
        mma_wait2();
      }
      // ---- dG_window = A_blend^T dz0 (dz0 is in h_1's tile), one pass per window
      const int nwin = (ktot + kKW - 1) / kKW;
      for (int wi = 0; wi < nwin; ++wi) {
        const int w0 = wi * kKW;
        if (nwin > 1) {  // rebuild this window's table and A rows
          if (wi > 0) ptx::bar_sync(bar_id, 128);
          fill_table(w0, false);
          scatter_a(w0);
          sync_for_mma();
        }
        if (tid < 32) {  // warp 0 issues (elected lane)
          ptx::tc_fence_after();
          for (int ks = 0; ks < 8; ++ks)
            ptx::mma_f16_ss_warp(tmem, ptx::smem_desc(sA + ks * 2 * kASbo, kASbo, 128, 0),
                            ptx::smem_desc(hT(1) + ks * 2 * kHSbo, kHSbo, 128, 0), id_dg, ks > 0 ? 1u : 0u);
          ptx::mma_commit_warp(&sh->mbar[g]);
        }
        mma_wait();
        ptx::bar_sync(bar_id, 128);  // the table is complete (nwin == 1: written in forward)
        const int kp = min(kKW, ktot - w0);
        const int texel = tid < kp ? sh->coltex[g][tid] : -1;
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          uint32_t vv[32];
          ptx::tmem_ld32(tmem_row + 32 * hh, vv);
          ptx::tmem_ld_wait();
          if (texel >= 0) {
            float *dst = dG + (size_t)texel * kHD + 32 * hh;
#pragma unroll
            for (int c = 0; c < 8; ++c)
              red_add_v4(dst + 4 * c, __uint_as_float(vv[4 * c]), __uint_as_float(vv[4 * c + 1]),
                         __uint_as_float(vv[4 * c + 2]), __uint_as_float(vv[4 * c + 3]));
          }
        }
        ptx::tc_fence_before();
      }
      if (stop_after) alive = false;
      if (!ptx::bar_red_or(bar_id, 128, alive)) break;  // every ray of the patch stopped
      ptx::bar_sync(bar_id, 128);  // TMEM reads and table reads done before the next chunk
    }
  }

  // ---- all groups done: add the TMEM dW^T / db accumulators to the caller's buffers
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  {
    const int f = tid;  // TMEM lane = input feature (64 = the bias row)
    for (int l = 1; l < L; ++l) {
      const bool head = l == L - 1;
      const int nout = head ? 4 : kHD;
      const uint32_t dcol = tmem_dw + lane_off + (uint32_t)((l - 1) * kHD);
      for (int h0 = 0; h0 < (head ? 16 : kHD); h0 += 16) {
        uint32_t vv[16];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
            "%11, %12, %13, %14, %15}, [%16];"
            : "=r"(vv[0]), "=r"(vv[1]), "=r"(vv[2]), "=r"(vv[3]), "=r"(vv[4]), "=r"(vv[5]),
              "=r"(vv[6]), "=r"(vv[7]), "=r"(vv[8]), "=r"(vv[9]), "=r"(vv[10]), "=r"(vv[11]),
              "=r"(vv[12]), "=r"(vv[13]), "=r"(vv[14]), "=r"(vv[15])
            : "r"(dcol + (uint32_t)h0)
            : "memory");
        ptx::tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const int o = h0 + e;
          if (o >= nout) continue;
          const float val = __uint_as_float(vv[e]);
          if (f < kHD) atomicAdd(Gp.dW[l] + (size_t)o * kHD + f, val);
          else if (f == kHD) atomicAdd(Gp.db[l] + o, val);
        }
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(sh->tmem_base, 512);
  }
}

// ------------------------------------------------------------------ K2 / K3
// dF_t[c] += sum_o dG_t[o] W0[o][cofs + c]: one warp per texel, W0 block in smem (fp32)
__global__ void __launch_bounds__(256)
    bwd_df_kernel(const float *__restrict__ dG, const __nv_bfloat16 *__restrict__ W0, int wstride,
                  int C, int R, int cat, float *__restrict__ dF) {
  extern __shared__ float sw[];  // [3 or 1][64][C]
  const int nblk = cat ? 3 : 1;
  for (int e = threadIdx.x; e < nblk * kHD * C; e += blockDim.x) {
    const int p = e / (kHD * C), rem = e - p * kHD * C, o = rem / C, c = rem - o * C;
    sw[e] = __bfloat162float(W0[(size_t)o * wstride + p * C + c]);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t ntex = (int64_t)3 * R * R;
  for (int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < ntex;
       t += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const float *w = sw + (cat ? (int)(t / ((int64_t)R * R)) : 0) * kHD * C;
    const float g0 = dG[t * kHD + lane], g1 = dG[t * kHD + 32 + lane];
    for (int c0 = 0; c0 < C; c0 += 32) {
      const int c = c0 + lane;
      float a = 0.0f;
#pragma unroll 8
      for (int o = 0; o < 32; ++o) {
        const float x0 = __shfl_sync(0xffffffffu, g0, o), x1 = __shfl_sync(0xffffffffu, g1, o);
        if (c < C) a += x0 * w[o * C + c] + x1 * w[(o + 32) * C + c];
      }
      if (c < C) dF[t * C + c] += a;
    }
  }
}

// dW0[o][cofs + c] += sum_t dG_t[o] F_t[c];  db0[o] += bscale sum_t dG_t[o] (+ the bias
// row).  A block reduces a slice of one plane's texels; thread c (< C + 1; column C is the
// bias, F := bscale) accumulates the 64 outputs of its column over the slice, reading the
// staged dG rows as shared-memory broadcasts.
constexpr int kWgTex = 32;
template <bool FP8>
__global__ void __launch_bounds__(288)
    bwd_dw0_kernel(const float *__restrict__ dG, const void *__restrict__ Fv, float fscale, int C,
                   int R, int cat, int wstride, float bscale, int bias_row, float *__restrict__ dW0,
                   float *__restrict__ db0, int tex_per_block) {
  __shared__ float4 sg[kWgTex][kHD / 4];
  const int c = threadIdx.x;
  const int64_t RR = (int64_t)R * R;
  const int64_t ntex = 3 * RR;
  const int64_t t0 = (int64_t)blockIdx.x * tex_per_block;
  const int64_t t1 = min(ntex, t0 + tex_per_block);
  const int plane = (int)(t0 / RR);  // tex_per_block divides R*R: one plane per block
  float acc[kHD];
#pragma unroll
  for (int o = 0; o < kHD; ++o) acc[o] = 0.0f;
  for (int64_t tb = t0; tb < t1; tb += kWgTex) {
    const int nt = (int)min((int64_t)kWgTex, t1 - tb);
    __syncthreads();
    for (int e = threadIdx.x; e < nt * (kHD / 4); e += blockDim.x)
      sg[e / (kHD / 4)][e % (kHD / 4)] = reinterpret_cast<const float4 *>(dG + (tb + e / (kHD / 4)) * kHD)[e % (kHD / 4)];
    __syncthreads();
    if (c <= C) {
      for (int tt = 0; tt < nt; ++tt) {
        float fv = bscale;
        if (c < C) {
          if constexpr (FP8) {
            const __half_raw hr = __nv_cvt_fp8_to_halfraw(
                static_cast<const __nv_fp8_storage_t *>(Fv)[(tb + tt) * C + c], __NV_E4M3);
            fv = fscale * __half2float(__half(hr));
          } else {
            fv = __bfloat162float(static_cast<const __nv_bfloat16 *>(Fv)[(tb + tt) * C + c]);
          }
        }
#pragma unroll
        for (int o4 = 0; o4 < kHD / 4; ++o4) {
          const float4 gv = sg[tt][o4];
          acc[4 * o4] += gv.x * fv;
          acc[4 * o4 + 1] += gv.y * fv;
          acc[4 * o4 + 2] += gv.z * fv;
          acc[4 * o4 + 3] += gv.w * fv;
        }
      }
    }
  }
  const int cofs = cat ? plane * C : 0;
  if (c < C) {
#pragma unroll
    for (int o = 0; o < kHD; ++o) atomicAdd(dW0 + (size_t)o * wstride + cofs + c, acc[o]);
  } else if (c == C && bscale != 0.0f) {
#pragma unroll
    for (int o = 0; o < kHD; ++o) atomicAdd(db0 + o, acc[o]);
  }
  if (blockIdx.x == 0 && bias_row && threadIdx.x < kHD) atomicAdd(db0 + threadIdx.x, dG[ntex * kHD + threadIdx.x]);
}

template <int NG>
static cudaError_t launch_bwd_k1(const RenderParams &P, const GradParams &Gp, float *dG, int sms,
                                 int64_t npatch, cudaStream_t st) {
  const size_t s1 = bw_smem_bytes<NG>(P.L) - sizeof(BwShared<NG>);  // dynamic part
  cudaError_t e = cudaFuncSetAttribute(render_bwd_tc_kernel<NG>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s1);
  if (e != cudaSuccess) return e;
  int grid = sms;
  if ((int64_t)grid * NG > npatch) grid = (int)((npatch + NG - 1) / NG);
  render_bwd_tc_kernel<NG><<<grid, 128 * NG, s1, st>>>(P, Gp, dG);
  return cudaGetLastError();
}

cudaError_t launch_render_backward_tc(const RenderParams &P0, const GradParams &Gp, cudaStream_t st) {
  if (P0.ray_end <= P0.ray_begin) return cudaSuccess;
  if (!P0.ws) return cudaErrorInvalidValue;
  RenderParams P = P0;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int R = P.R, C = P.C;
  const int64_t ntex = (int64_t)3 * R * R;
  float *dG = reinterpret_cast<float *>(static_cast<uint8_t *>(P.ws) +
                                        ((tc_workspace_bytes(R, kHD) + 255) & ~size_t(255)));
  cudaError_t e = cudaMemsetAsync(dG, 0, (size_t)(ntex + 1) * kHD * 4, st);
  if (e != cudaSuccess) return e;
  e = launch_preproject(P, st);  // G = F W0^T + bscale b0, patch counter = 0
  if (e != cudaSuccess) return e;
  const int64_t HW = (int64_t)P.H * P.W;
  const int nv = (int)((P.ray_end - 1) / HW - P.ray_begin / HW + 1);
  const int64_t npatch = (int64_t)nv * ((P.H + 3) / 4) * ((P.W + 3) / 4);
  timer_begin(P.timer, st);
  const bool ng2 = bw_smem_bytes<2>(P.L) <= kSmemLimit && 2 * (kHD + (P.L - 2) * kHD + 16 + 48) <= 512;
  e = ng2 ? launch_bwd_k1<2>(P, Gp, dG, sms, npatch, st) : launch_bwd_k1<1>(P, Gp, dG, sms, npatch, st);
  timer_end(P.timer, st);
  if (e != cudaSuccess) return e;
  // K2: dF = dG W0 (per plane block for concat); K3: dW0, db0
  const bool cat = P.agg == 2;
  const int wstride = cat ? 3 * C : C;
  const __nv_bfloat16 *W0 = reinterpret_cast<const __nv_bfloat16 *>(P.w[0]);
  const size_t s2 = (size_t)(cat ? 3 : 1) * kHD * C * 4;
  e = cudaFuncSetAttribute(bwd_df_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s2);
  if (e != cudaSuccess) return e;
  int g2 = (int)((ntex * 32 + 255) / 256);
  if (g2 > sms * 2) g2 = sms * 2;  // W0 block staged once per block
  bwd_df_kernel<<<g2, 256, s2, st>>>(dG, W0, wstride, C, R, cat ? 1 : 0, Gp.dF);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  // texels per K3 block: a divisor of R*R near R*R*3/(2 sms)
  const int64_t RR = (int64_t)R * R;
  int tpb = (int)((3 * RR + 2 * sms - 1) / (2 * sms));
  while (RR % tpb) ++tpb;
  const float bscale = P.smode != 0 ? 0.0f : (P.agg == 0 ? 1.0f : (1.0f / 3.0f));
  const int nthr = ((C + 1) + 31) / 32 * 32;  // one thread per column of dW0 (+ the bias)
  (P.tp_fp8 ? bwd_dw0_kernel<true> : bwd_dw0_kernel<false>)<<<(int)((3 * RR) / tpb), nthr, 0, st>>>(
      dG, P.tp, P.tp_scale, C, R, cat ? 1 : 0, wstride, bscale,
      P.smode != 0 ? 1 : 0, Gp.dW[0], Gp.db[0], tpb);
  return cudaGetLastError();
}

}  // namespace dmv3d
