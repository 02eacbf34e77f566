// render_tc.cu -- the tcgen05/TMEM renderer engine (DMV3D_ENGINE_TCGEN05).
//
// Design:
//  * K0 `preproject`: by linearity of the first MLP layer, the triplane is
//    pre-multiplied by W0 once per denoise step, G = F W0^T + b0, stored
//    fp16 channels-last [3][R][R][HD] in the caller's workspace (1.5 MiB
//    at R=64, HD=64).  Decoding a sample then needs the bilinear blend of G
//    (= W0 h0 + b0, exact in real arithmetic).
//  * K1 `render_tc`: persistent, one CTA per SM, NG independent groups of 4
//    warps.  A group marches a 4x4 pixel patch (16 rays) in chunks of 8
//    samples: tile = 128 rows = 16 rays x 8 samples = the 128 TMEM lanes.
//    Per chunk:
//      1. each row computes its sample point and texel cells (bit-exact
//         fp32 geometry, rows a1-a3);
//      2. the group reduces the per-axis texel ranges (REDUX) into a small
//         bounding box per plane, and stages those texels of G in shared
//         memory with 16-byte cp.async (SWIZZLE_128B MN-major B operand);
//      3. each row writes its 12 bilinear weights (x 1/3 for the mean) into
//         a sparse fp16 A row, and one tcgen05.mma chain computes
//         D = A . G_tile = W0 h0 + b0 for all 128 samples (the blend runs on
//         the tensor cores, each staged texel is read once per tile);
//      4. the remaining MLP layers run as tcgen05.mma with fp16 activations
//         written back by the row threads (ReLU + pack in one cvt), weights
//         resident in shared memory, biases folded in as an extra K column,
//         fp32 accumulation in TMEM; the 4-wide head is an N=16 MMA;
//      5. sigma/rgb are composited with an 8-lane shuffle scan per ray, the
//         ray stops once T < term_eps, and the ray epilogue applies the DDIM
//         update (row a6).
//    The NG groups interleave on the SM: while one group waits on its MMA
//    chain the others stage, scatter and run epilogues.
#include <cuda_fp16.h>
#include <cuda_fp8.h>

#include "common.cuh"
#include "kernels.h"
#include "tc_ptx.cuh"

namespace dmv3d {

// Phase timing (tools/phases.py builds the library with -DDMV3D_PHASES): every thread
// accumulates clock64 deltas per phase; each group's row 0 adds them to counters[8..15].
#ifdef DMV3D_PHASES
#define PH_DECL                                            \
  unsigned long long ph_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0}; \
  long long ph_t = clock64();
#define PH(i)                         \
  do {                                \
    const long long ph_n = clock64(); \
    ph_acc[i] += ph_n - ph_t;         \
    ph_t = ph_n;                      \
  } while (0)
#else
#define PH_DECL
#define PH(i) \
  do {        \
  } while (0)
#endif

constexpr int kTcHD = 64;       // hidden width of the tensor-core engine
constexpr int kTcKMax = 128;    // max staged texels (K) per MMA pass
constexpr int kPatch = 4;       // 4x4 rays per patch
constexpr int kChunk = 8;       // samples per ray per tile
constexpr int kGridKZ = 4;      // density grid: 8x4x4 point blocks per patch column (chunks)
constexpr uint32_t kHeadAlt = 112;  // second head accumulator: spare TMEM columns of a group
constexpr uint32_t kWsHeader = kTcWsHeader;

// shared-memory carve-up (bytes)
// sparse A tile, K-major SWIZZLE_NONE: 8-row groups SBO = 2048 + 32 bytes apart, so rows
// m, m+8, m+16, m+24 of a warp fall into different banks (the 2-byte weight scatter)
constexpr uint32_t kASbo = (kTcKMax / 8) * 128 + 32;   // 2080
constexpr uint32_t kATileBytes = 16 * kASbo;           // 32.5 KiB (NG of them keep 1 KiB alignment)
constexpr uint32_t kBTileBytes = kTcKMax * kTcHD * 2;  // 16 KiB, 128 B per texel row
constexpr uint32_t kWK = kTcHD + 16;                   // weights K incl. bias column
constexpr uint32_t kWSbo = (kWK / 8) * 128;            // 1280
constexpr uint32_t kWHidden = kTcHD * kWK * 2;         // 10 KiB per hidden layer
constexpr uint32_t kWHead = 16 * kWK * 2;              // 2.5 KiB
constexpr size_t kSmemLimit = 232448;                  // 227 KiB per CTA

// header (patch counter) + G [3 R R + 1][HD]: the last row holds b0 for the
// half-pixel mode's bias column
size_t tc_workspace_bytes(int R, int HD, int assets) {
  return kWsHeader + (size_t)assets * ((size_t)3 * R * R + 1) * HD * 2;
}

// C = channels per plane (the MLP input is 3 C for the concat aggregation)
bool tc_supported(int C, int HD, int L) {
  return HD == kTcHD && C >= 8 && C <= 256 && C % 8 == 0 && L >= 2 && L <= kMaxLayers;
}

template <int NG>
struct TcShared {
  uint64_t mbar[NG];
  uint32_t tmem_base;
  int patch[NG];
  int bbox[NG][2][8];  // per chunk parity: xmin,ymin,zmin,-,xmax,ymax,zmax,-
  int coltex[NG][kTcKMax];  // staged column -> texel index of G (-1: zero fill)
  float head_bias[4];
  unsigned n_tiles[NG], n_kcols[NG];  // blend windows issued, staged K columns (counters[4..5])
};

// dynamic shared memory of the render kernel (tiles + weights); the TcShared block is a
// static __shared__ variable (so its accesses compile to LDS/STS/ATOMS, not generic ones)
template <int NG>
static size_t tc_smem_bytes(int L) {
  // the B tiles follow the NG A tiles and must stay 1 KiB aligned (SWIZZLE_128B atoms)
  static_assert((NG * kATileBytes) % 1024 == 0, "A tiles must keep the B tiles 1 KiB aligned");
  return 1024 /*align slack*/ + (size_t)NG * (kATileBytes + kBTileBytes) +
         (size_t)(L - 2) * kWHidden + kWHead;
}

// ------------------------------------------------------------------ K0
// G[t][o] = fp16(sum_c F[t][c] W0[o][c] + b0[o] * bscale); one warp per 4 texels (bf16;
// per texel for FP8), lane -> outputs (2 lane, 2 lane + 1); W0 transposed in smem
// (conflict-free), each of its elements read once per 4 texels.
// W0 rows have stride `wstride` (3 C for the concat aggregation, whose planes are
// projected by their own column block of W0).  Optionally zeroes the patch counter
// and writes fp16(b0) to `gbias` (the bias row of the half-pixel mode).
// FP8: F is E4M3 storage (row f4) dequantised by `fscale`; 16 channels per 16-B load.
template <bool FP8>
__global__ void __launch_bounds__(256)
    preproject_kernel(const void *__restrict__ Fv, int ntex, int C, int wstride,
                      const __nv_bfloat16 *__restrict__ W0, const float *__restrict__ b0,
                      float bscale, float fscale, __half *__restrict__ G, unsigned int *counter,
                      __half *__restrict__ gbias, int64_t per_asset, int assets,
                      unsigned int *range_flags) {
  extern __shared__ __align__(16) float2 swt[];  // [C][HD/2] (o pairs)
  for (int e = threadIdx.x; e < kTcHD * C; e += blockDim.x) {  // o fastest: conflict-free stores
    const int c = e / kTcHD, o = e - c * kTcHD;
    reinterpret_cast<float *>(swt)[c * kTcHD + o] = __bfloat162float(W0[(size_t)o * wstride + c]);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && counter) *counter = 0u;
  if (blockIdx.x == 0 && gbias)  // every asset's bias row (G block row per_asset)
    for (int e = threadIdx.x; e < assets * kTcHD; e += blockDim.x)
      gbias[(int64_t)(e / kTcHD) * (per_asset + 1) * kTcHD + e % kTcHD] =
          __float2half_rn(__ldg(b0 + e % kTcHD));
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const float bias0 = __ldg(b0 + 2 * lane) * bscale, bias1 = __ldg(b0 + 2 * lane + 1) * bscale;
  const int64_t w_first = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t w_step = ((int64_t)gridDim.x * blockDim.x) >> 5;
  // stores G[t] (this lane's output pair), with the fp16 range guard: G outside +-65504
  // (or NaN) raises range flag bit 0; the value is stored as inf / NaN (no silent clamp)
  auto store = [&](int64_t t, float a0, float a1) {
    if (!(fabsf(a0) <= 65504.0f && fabsf(a1) <= 65504.0f)) atomicOr(range_flags, 1u);
    const int64_t ta = t / per_asset;  // asset: its G block has one extra (bias) row
    reinterpret_cast<uint32_t *>(G + (t + ta) * kTcHD)[lane] = ptx::pack_f16x2(a0, a1);
  };
  if constexpr (FP8) {
    for (int64_t t = w_first; t < ntex; t += w_step) {
      const uint4 *src = reinterpret_cast<const uint4 *>(static_cast<const uint8_t *>(Fv) + t * C);
      float s0 = 0.0f, s1 = 0.0f;
      for (int q = 0; q < C / 16; ++q) {
        const uint4 u = __ldg(src + q);
        const uint32_t uv[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int e = 0; e < 8; ++e) {  // e4m3 pairs -> half2 (exact) -> float
          const __half2_raw hr = __nv_cvt_fp8x2_to_halfraw2(
              (__nv_fp8x2_storage_t)((uv[e >> 1] >> (16 * (e & 1))) & 0xffffu), __NV_E4M3);
          const float2 f = __half22float2(*reinterpret_cast<const __half2 *>(&hr));
          const float2 w0 = swt[(q * 16 + 2 * e) * (kTcHD / 2) + lane];
          const float2 w1 = swt[(q * 16 + 2 * e + 1) * (kTcHD / 2) + lane];
          s0 += w0.x * f.x + w1.x * f.y;
          s1 += w0.y * f.x + w1.y * f.y;
        }
      }
      store(t, bias0 + fscale * s0, bias1 + fscale * s1);
    }
  } else {
    // bf16: a warp projects kTexW texels per iteration, so every W0 element it reads from
    // shared memory serves kTexW texels (shared-memory bound otherwise); lane q holds
    // 16-B chunk q of each texel row (C <= 256: <= 32 chunks), read by shuffle
    constexpr int kTexW = 4;
    const int nq = C / 8;
    const __nv_bfloat16 *F = static_cast<const __nv_bfloat16 *>(Fv);
    for (int64_t tg = w_first; tg * kTexW < ntex; tg += w_step) {
      uint4 cur[kTexW];
#pragma unroll
      for (int u = 0; u < kTexW; ++u) {
        const int64_t t = tg * kTexW + u;
        cur[u] = (t < ntex && lane < nq) ? __ldg(reinterpret_cast<const uint4 *>(F + t * C) + lane)
                                         : make_uint4(0u, 0u, 0u, 0u);
      }
      float a0[kTexW], a1[kTexW];
#pragma unroll
      for (int u = 0; u < kTexW; ++u) a0[u] = a1[u] = 0.0f;
      for (int q = 0; q < nq; ++q) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 w0 = swt[(q * 8 + 2 * e) * (kTcHD / 2) + lane];
          const float2 w1 = swt[(q * 8 + 2 * e + 1) * (kTcHD / 2) + lane];
#pragma unroll
          for (int u = 0; u < kTexW; ++u) {
            const uint32_t word = __shfl_sync(0xffffffffu, e == 0 ? cur[u].x : e == 1 ? cur[u].y
                                                           : e == 2 ? cur[u].z : cur[u].w, q);
            const float f0 = bf16lo(word), f1 = bf16hi(word);
            a0[u] += w0.x * f0 + w1.x * f1;
            a1[u] += w0.y * f0 + w1.y * f1;
          }
        }
      }
#pragma unroll
      for (int u = 0; u < kTexW; ++u) {
        const int64_t t = tg * kTexW + u;
        if (t < ntex) store(t, bias0 + a0[u], bias1 + a1[u]);
      }
    }
  }
}

// ------------------------------------------------------------------ K1
__device__ __forceinline__ uint32_t a_row(int m) {
  return (uint32_t)((m >> 3) * kASbo + (m & 7) * 16);
}
// byte offset of column k in a row: (k >> 3) * 128 + (k & 7) * 2 == 2 k + 112 (k >> 3)
// (k >= 0): a shift and two multiply-adds instead of shift / mask / or chains
__device__ __forceinline__ uint32_t a_col(int k) { return (uint32_t)(2 * k + 112 * (k >> 3)); }

// hidden activation (reading A5) -> fp16 pair; ReLU folds into the conversion, SiLU and
// softplus are evaluated in fp32 (fast-math exp / log, within the tensor-core tolerance)
template <int ACT>
__device__ __forceinline__ uint32_t pack_act(float lo, float hi) {
  if constexpr (ACT == 1) {
    return ptx::pack_f16x2(__fdividef(lo, 1.0f + __expf(-lo)), __fdividef(hi, 1.0f + __expf(-hi)));
  } else if constexpr (ACT == 2) {
    return ptx::pack_f16x2(fmaxf(lo, 0.0f) + __logf(1.0f + __expf(-fabsf(lo))),
                           fmaxf(hi, 0.0f) + __logf(1.0f + __expf(-fabsf(hi))));
  } else {
    return ptx::pack_relu_f16x2_inf(lo, hi);
  }
}

// epilogue of one MLP layer: accumulator row (HD fp32 TMEM columns at `d_row`) ->
// activation -> fp16 pairs -> the next layer's A operand in TMEM at `a_row` (HD/2
// columns).  The bias K block that follows it (k = HD: 1.0, k = HD+1..HD+15: 0) is
// constant and written once per kernel.
template <int ACT>
__device__ __forceinline__ void act_epilogue(uint32_t d_row, uint32_t a_row) {
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    uint32_t v[32];
    ptx::tmem_ld32(d_row + 32 * h, v);
    ptx::tmem_ld_wait();
    uint32_t pk[16];
    const float *f = reinterpret_cast<const float *>(v);
#pragma unroll
    for (int e = 0; e < 16; ++e) pk[e] = pack_act<ACT>(f[2 * e], f[2 * e + 1]);
    ptx::tmem_st16(a_row + 16 * h, pk);
  }
  ptx::tmem_st_wait();
}

// GRID = false: the renderer (rays, compositing, DDIM epilogue).  GRID = true: the
// density grid (row f3): a "patch" is an 8x4x4 block of grid points, decoded in one
// 128-row tile through the same staged-texel blend + MLP MMAs.
template <int NG, bool GRID, int ACT>
__global__ void __launch_bounds__(128 * NG, 1)
    render_tc_kernel(const __grid_constant__ RenderParams P) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~uintptr_t(1023));
  uint8_t *tileA0 = smem;
  uint8_t *tileB0 = smem + NG * kATileBytes;
  uint8_t *wsm = tileB0 + NG * kBTileBytes;
  const int L = P.L;
  __shared__ TcShared<NG> sh_s;
  TcShared<NG> *sh = &sh_s;

  const int tid_cta = threadIdx.x;
  // warp index through a shuffle: ptxas then knows it (and the group, the group's TMEM
  // columns, tile addresses and MMA descriptors derived from it) is warp-uniform and keeps
  // them in uniform registers -- no R2UR per MMA issue
  const int warp = __shfl_sync(0xffffffffu, tid_cta >> 5, 0);
  const int g = warp >> 2;        // group
  const int tid = tid_cta & 127;  // row within the group's tile
  const int bar_id = 1 + g;

  // ---- prologue: barriers, TMEM, weights (fp16, K-major, bias column)
  if (tid_cta == 0) {
    for (int i = 0; i < NG; ++i) {
      ptx::mbar_init(&sh->mbar[i], 1);
      sh->n_tiles[i] = sh->n_kcols[i] = 0u;
    }
    for (int i = 0; i < NG; ++i)
      for (int p = 0; p < 2; ++p)
        for (int e = 0; e < 8; ++e) sh->bbox[i][p][e] = (e < 4) ? 0x7fffffff : -1;
    ptx::fence_mbar_init();
  }
  constexpr uint32_t kCols = NG * 2 * kTcHD;  // per group: accumulator + fp16 A operand
  constexpr uint32_t kTmemCols = kCols <= 32 ? 32 : kCols <= 64 ? 64 : kCols <= 128 ? 128
                                 : kCols <= 256 ? 256 : 512;
  if (warp == 0) ptx::tmem_alloc(&sh->tmem_base, kTmemCols);
  for (int l = 1; l < L; ++l) {
    const int nout = (l == L - 1) ? 16 : kTcHD;
    const int nreal = (l == L - 1) ? 4 : kTcHD;
    uint8_t *wl = wsm + (l - 1) * kWHidden;
    const __nv_bfloat16 *W = reinterpret_cast<const __nv_bfloat16 *>(P.w[l]);
    for (int e = tid_cta; e < nout * (int)kWK; e += 128 * NG) {
      const int n = e / kWK, k = e - n * kWK;
      float v = 0.0f;
      if (n < nreal) {
        if (k < kTcHD) v = __bfloat162float(W[n * kTcHD + k]);
        else if (k == kTcHD) v = __ldg(P.b[l] + n);
      }
      const uint32_t off = (n >> 3) * kWSbo + (k >> 3) * 128 + (n & 7) * 16 + (k & 7) * 2;
      *reinterpret_cast<__half *>(wl + off) = __float2half_rn(v);
    }
  }
  if (tid_cta < 4) sh->head_bias[tid_cta] = __ldg(P.b[L - 1] + tid_cta);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  // TMEM base through a shuffle: warp-uniform (uniform registers in the MMA issue)
  const uint32_t tmem = __shfl_sync(0xffffffffu, sh->tmem_base, 0) + (uint32_t)(g * 2 * kTcHD);
  const uint32_t tmem_row = tmem + ((uint32_t)((warp & 3) * 32) << 16);
  {  // the activation operand's bias K block ([1, 0 x 15] per row) is constant: once
    const uint32_t bias[8] = {0x3C00u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
    ptx::tmem_st8(tmem_row + kTcHD + kTcHD / 2, bias);
    ptx::tmem_st_wait();
  }

  // tile addresses from a warp-uniform (shuffled) 32-bit base: ptxas keeps them and the
  // descriptor words built from them in uniform registers
  const uint32_t sbase = __shfl_sync(0xffffffffu, ptx::smem_u32(tileA0), 0);
  const uint32_t sA = sbase + (uint32_t)(g * kATileBytes);
  const uint32_t sB = sbase + (uint32_t)(NG * kATileBytes + g * kBTileBytes);
  const uint32_t sW = sbase + (uint32_t)(NG * (kATileBytes + kBTileBytes));
  // low descriptor words of each operand's first K step (start address >> 4 | LBO >> 4
  // << 16); a K step adds its byte offset >> 4 (no carry out of the 14-bit field)
  const uint32_t a_lo0 = ((sA >> 4) & 0x3FFFu) | ((128u >> 4) << 16);
  const uint32_t b_lo0 = ((sB >> 4) & 0x3FFFu) | ((1024u >> 4) << 16);
  const uint32_t w_lo0 = ((sW >> 4) & 0x3FFFu) | ((128u >> 4) << 16);
  constexpr uint64_t a_hi = ((uint64_t)(kASbo >> 4) << 32) | (1ull << 46);
  constexpr uint64_t b_hi = ((uint64_t)(1024u >> 4) << 32) | (1ull << 46) | (2ull << 61);
  constexpr uint64_t w_hi = ((uint64_t)(kWSbo >> 4) << 32) | (1ull << 46);
  const uint32_t sArow = sA + a_row(tid);
  constexpr uint32_t idesc_blend = ptx::idesc_f16(128, kTcHD, 1);
  constexpr uint32_t idesc_hidden = ptx::idesc_f16(128, kTcHD, 0);
  constexpr uint32_t idesc_head = ptx::idesc_f16(128, 16, 0);

  const __half *G0 = reinterpret_cast<const __half *>(reinterpret_cast<const uint8_t *>(P.tp) +
                                                       kWsHeader);
  const int64_t g_stride = ((int64_t)3 * P.R * P.R + 1) * kTcHD;  // per asset (batched launches)
  const __half *G = G0;
  unsigned int *counter = reinterpret_cast<unsigned int *>(const_cast<void *>(P.tp));

  // patch space: views [v_lo, v_hi] of the ray range, 4x4 patches
  const int64_t HW = (int64_t)P.H * P.W;
  const int v_lo = (int)(P.ray_begin / HW);
  const int v_hi = (int)((P.ray_end - 1) / HW);
  const int PH = (P.H + kPatch - 1) / kPatch, PW = (P.W + kPatch - 1) / kPatch;
  // density grid: a "patch" is a column of kGridKZ blocks of 8x4x4 points along z, walked
  // as chunks so the next block's staging overlaps the current block's MLP
  const int GB[3] = {(P.grid_res + 7) / 8, (P.grid_res + 3) / 4,
                     (P.grid_res + 4 * kGridKZ - 1) / (4 * kGridKZ)};
  // interleaved ray tiles (§8e): the work queue enumerates this rank's tiles' patches
  const int TP = P.tile_size / kPatch;  // patches per tile side (0: no tiling)
  int64_t tile_first = 0, tile_n = 0;
  if (!GRID && TP > 0)
    owned_tiles(v_lo, v_hi, P.H, P.W, P.tile_size, P.tile_rank, P.tile_count, tile_first, tile_n);
  const int64_t TH = TP > 0 ? (P.H + P.tile_size - 1) / P.tile_size : 1;
  const int64_t TW = TP > 0 ? (P.W + P.tile_size - 1) / P.tile_size : 1;
  const int64_t npatch = GRID ? (int64_t)GB[0] * GB[1] * GB[2]
                              : TP > 0 ? tile_n * TP * TP : (int64_t)(v_hi - v_lo + 1) * PH * PW;
  const int slot = tid >> 3, q = tid & 7;
  const int R = P.R;
  const float wscale = (P.agg == 0) ? (1.0f / 3.0f) : 1.0f;
  // half-pixel zero padding: the blend weights of a sample no longer sum to one per
  // plane, so b0 is not folded into G but added by one extra A column (weight 1)
  // that reads the bias row G[3 R R]
  const int hb = P.smode != 0 ? 1 : 0;
  // geometry fast path (uniform): align-corners sampling with power-of-two box extents
  const bool fastgeo = P.smode == 0 && P.inv_ext[0] != 0.0f && P.inv_ext[1] != 0.0f && P.inv_ext[2] != 0.0f;
  const float rm1 = __int2float_rn(R - 1);

  uint32_t mphase = 0;
  unsigned n_hit = 0, n_samples = 0, n_term = 0, n_rays = 0;  // per thread: fits 32 bits
  unsigned n_range = 0;  // samples whose head output is not finite (fp16 overflow upstream)
  PH_DECL
  int chunk_ctr = 0;

  // column -> texel table of the tile's window [w0, w0 + kpad) (one column per thread);
  // `bb` = the chunk's per-axis texel ranges (min at [0..2], max at [4..6]).  `direct`:
  // thread kl also copies texel row kl into the B tile itself (8 cp.async, 16-B chunks
  // XOR-swizzled by the row: the SWIZZLE_128B MN-major layout), so the prefetch needs no
  // table round trip and no second barrier.  (Writing the table in that case too is dead
  // but measured faster than dropping it: 2.89 vs 3.05 ms per cfg3 step.)
  auto fill_table = [&](const int *bb, int w0, bool direct) {
    const int lo0 = bb[0], lo1 = bb[1], lo2 = bb[2];
    const int ext0 = bb[4] - lo0 + 2, ext1 = bb[5] - lo1 + 2, ext2 = bb[6] - lo2 + 2;
    const int base1 = ext0 * ext1, base2 = base1 + ext0 * ext2;
    const int ktex = base2 + ext1 * ext2;
    const int ktot = ktex + hb;
    const int kpad = (min(kTcKMax, ktot - w0) + 15) & ~15;
    // column col = tid + 64 (mod 128): a window of <= 64 columns is staged by warps 2-3,
    // keeping warp 0 (the MMA issuer, the group's critical warp) and warp 1 free
    const int col = (tid + 64) & 127;
    if (col < kpad) {
      const int kg = w0 + col;
      int texel = -1;
      if (kg == ktex && hb) {
        texel = 3 * R * R;
      } else if (kg < ktex) {
        int loc, bw, ta0, tb0, pl;
        if (kg >= base2) { pl = 2; loc = kg - base2; bw = ext1; ta0 = lo1; tb0 = lo2; }
        else if (kg >= base1) { pl = 1; loc = kg - base1; bw = ext0; ta0 = lo0; tb0 = lo2; }
        else { pl = 0; loc = kg; bw = ext0; ta0 = lo0; tb0 = lo1; }
        // row = floor(loc / bw): loc < 2^13 and bw < 2^8, so an approximate
        // reciprocal is never off by one
        const int rr = (int)(((float)loc + 0.5f) * __fdividef(1.0f, (float)bw));
        texel = (pl * R + tb0 + rr) * R + ta0 + (loc - rr * bw);
      }
      sh->coltex[g][col] = texel;
      if (direct) {  // this thread stages texel row col itself: no table round trip
        const uint32_t drow = sB + (uint32_t)(col << 7);
        const __half *src = G + (size_t)max(texel, 0) * kTcHD;
        const uint32_t nb = texel >= 0 ? 16u : 0u;
#pragma unroll
        for (int ch = 0; ch < 8; ++ch)
          ptx::cp_async16(drow + (uint32_t)((ch ^ (col & 7)) << 4), src + ch * 8, nb);
      }
    }
  };
  // cp.async the window's texels of G into the B tile: 8 threads per 128-B texel row,
  // SWIZZLE_128B (16-B chunk index XOR row index within each 1 KiB atom)
  auto stage = [&](const int *bb, int w0) {
    const int e0 = bb[4] - bb[0] + 2, e1 = bb[5] - bb[1] + 2, e2 = bb[6] - bb[2] + 2;
    const int ktot = e0 * e1 + e0 * e2 + e1 * e2 + hb;
    const int kpad = (min(kTcKMax, ktot - w0) + 15) & ~15;
    for (int e = tid; e < kpad * 8; e += 128) {
      const int kl = e >> 3, ch = e & 7;
      const int texel = sh->coltex[g][kl];
      const uint32_t dst = sB + (uint32_t)((kl << 7) + ((ch ^ (kl & 7)) << 4));
      ptx::cp_async16(dst, G + (size_t)max(texel, 0) * kTcHD + ch * 8, texel >= 0 ? 16u : 0u);
    }
  };

  while (true) {
    if (tid == 127) sh->patch[g] = (int)atomicAdd(counter, 1u);  // warp 3: off the issuer
    ptx::bar_sync(bar_id, 128);
    const int64_t patch = sh->patch[g];
    if (patch >= npatch) break;
    PH(7);
    int v = 0, i = 0, j = 0;
    int64_t r = 0;
    bool pix;
    Ray ray;
    ray.hit = false;
    ray.t_near = ray.t_far = 0.0f;
    int gx = 0, gy = 0, gz0 = 0;  // GRID: this row's point column (x, y) and first z
    if constexpr (GRID) {
      const int G = P.grid_res;
      const int bx = (int)(patch % GB[0]), by = (int)((patch / GB[0]) % GB[1]),
                bz = (int)(patch / ((int64_t)GB[0] * GB[1]));
      gx = bx * 8 + (tid & 7);
      gy = by * 4 + ((tid >> 3) & 3);
      gz0 = bz * 4 * kGridKZ + (tid >> 5);
      pix = gx < G && gy < G;
      ray.hit = pix;
    } else {
      int prow, pcol;
      if (TP > 0) {  // k-th owned tile, w-th patch in it
        const int64_t tau = tile_first + (patch / (TP * TP)) * P.tile_count;
        const int w = (int)(patch % (TP * TP));
        v = (int)(tau / (TH * TW));
        const int64_t trem = tau % (TH * TW);
        prow = (int)(trem / TW) * TP + w / TP;
        pcol = (int)(trem % TW) * TP + w % TP;
      } else {
        v = v_lo + (int)(patch / ((int64_t)PH * PW));
        const int prem = (int)(patch % ((int64_t)PH * PW));
        prow = prem / PW;
        pcol = prem % PW;
      }
      i = prow * kPatch + (slot >> 2);
      j = pcol * kPatch + (slot & 3);
      G = G0 + (int64_t)(v / P.V_asset) * g_stride;  // this view's asset's projected triplane
      const int act = view_action(P, v);               // uniform over the patch
      if (act != 0) {  // not rendered: nothing, or x_{t-1} = x_t for a kept view
        if (act == 2 && q < 3 && i < P.H && j < P.W) {
          const int64_t rr = (int64_t)v * HW + (int64_t)i * P.W + j;
          if (rr >= P.ray_begin && rr < P.ray_end) copy_kept(P, v, i, j, q);
        }
        continue;
      }
      r = (int64_t)v * HW + (int64_t)i * P.W + j;
      pix = (i < P.H) && (j < P.W) && r >= P.ray_begin && r < P.ray_end;
      if (pix) ray = make_ray(P.intr, P.c2w, v, i, j, P.lo, P.hi);
      if (pix && P.plucker && q < 6) plucker_write(P.plucker, P.H, P.W, v, i, j, q, ray);
    }
    bool alive = pix && ray.hit;
    const float delta = alive ? sample_delta(ray, P.N) : 0.0f;
    float T = 1.0f, acc0 = 0.0f, acc1 = 0.0f, acc2 = 0.0f;
    if (q == 0) {
      n_rays += pix ? 1 : 0;
      n_hit += alive ? 1 : 0;
    }

    // Chunk pipeline: the geometry, texel window and cp.async staging of chunk
    // c+1 are issued while chunk c's MLP runs on the tensor cores (the staged B
    // tile is free once c's blend MMA has completed).  Chunk c+1 is prepared for
    // the rays alive before c's compositing; rays that terminate in c get zero A
    // rows in c+1.
    int ix[3] = {0, 0, 0};
    float wl[3] = {0.f, 0.f, 0.f}, wh[3] = {0.f, 0.f, 0.f};  // weights of texels ix, ix + 1
    int par = 0;
    // geometry + window + staging of window 0 for the chunk starting at kk (the
    // chunk's bbox slot must still hold its reset state when this runs)
    auto prefetch = [&](int kk, bool spec_alive) {
      par = chunk_ctr & 1;
      ++chunk_ctr;
      const int k = kk + q;
      // GRID: one point per row, z advancing 4 per chunk
      const bool sv = spec_alive && (GRID ? gz0 + (kk / kChunk) * 4 < P.grid_res : k < P.N);
      // rows without a sample keep the previous chunk's values: nothing reads them (the box
      // reduction masks them, the scatter skips them: a row live at the scatter was live here)
      if (sv) {
        float p[3];
        if constexpr (GRID) {
          const int id3[3] = {gx, gy, gz0 + (kk / kChunk) * 4};
          const float gm1 = __int2float_rn(P.grid_res - 1);
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            const float s = __fdiv_rn(__int2float_rn(id3[a]), gm1);
            p[a] = __fadd_rn(P.lo[a], __fmul_rn(s, __fsub_rn(P.hi[a], P.lo[a])));
          }
        } else {
          const float u = P.jitter ? jitter_u(P.seed, (uint64_t)r * P.N + k) : 0.5f;
          sample_p(ray, sample_t(ray, delta, k, u), p);
        }
        if (fastgeo) {  // align-corners mode, power-of-two box extents: texel_coord's
                        // multiply path with no per-axis branches (the same IEEE ops)
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
      // reset the other parity's slot for the next chunk (all its readers passed a barrier)
      if (tid >= 120) sh->bbox[g][par ^ 1][tid - 120] = (tid < 124) ? 0x7fffffff : -1;  // warp 3
      fill_table(sh->bbox[g][par], 0, true);
    };

    bool have = ptx::bar_red_or(bar_id, 128, alive);
    if (have) prefetch(0, alive);
    PH(0);
    for (int k0 = 0; have;) {
      const int k = k0 + q;
      const int gz = gz0 + (k0 / kChunk) * 4;  // GRID: this chunk's z
      const bool sv = alive && (GRID ? gz < P.grid_res : k < P.N);
      const int *bb = sh->bbox[g][par];
      const int lo0 = bb[0], lo1 = bb[1], lo2 = bb[2];
      const int ext0 = bb[4] - lo0 + 2, ext1 = bb[5] - lo1 + 2, ext2 = bb[6] - lo2 + 2;
      // plane p uses axes (a, b): XY (0,1), XZ (0,2), YZ (1,2); row-major bbox rows
      const int base1 = ext0 * ext1, base2 = base1 + ext0 * ext2;
      const int ktex = base2 + ext1 * ext2;
      const int ktot = ktex + hb;
      const int ca = ix[0] - lo0, cb = ix[1] - lo1, cc = ix[2] - lo2;
      const int cols[3] = {cb * ext0 + ca, base1 + cc * ext0 + ca, base2 + cc * ext1 + cb};
      const int bws[3] = {ext0, ext0, ext1};
      const float la[3] = {wl[0], wl[0], wl[1]}, ha[3] = {wh[0], wh[0], wh[1]};
      const float lb[3] = {wl[1], wl[2], wl[2]}, hb3[3] = {wh[1], wh[2], wh[2]};

      // ---- blend on the tensor cores: window 0 was staged by prefetch; rare extra
      //      windows (> kTcKMax texels) are staged synchronously
      for (int w0 = 0; w0 < ktot; w0 += kTcKMax) {
        const int kp = min(kTcKMax, ktot - w0);
        const int kpad = (kp + 15) & ~15;
        // zero the row's kpad columns: kpad / 16 iterations of two 16-B stores (a plain loop;
        // the compiler's multi-level unrolling of a one-store loop cost ~35 control
        // instructions per chunk)
#pragma unroll 1
        for (int kc = 0; kc < kpad / 16; ++kc) {
          ptx::sts128(sArow + (uint32_t)(kc << 8), 0u, 0u, 0u, 0u);
          ptx::sts128(sArow + (uint32_t)((kc << 8) + 128), 0u, 0u, 0u, 0u);
        }
        if (sv) {
#pragma unroll
          for (int pl = 0; pl < 3; ++pl) {
            const float gy = lb[pl] * wscale, fy = hb3[pl] * wscale;
            const int c0 = cols[pl] - w0, c2 = c0 + bws[pl];
            const float w4[4] = {la[pl] * gy, ha[pl] * gy, la[pl] * fy, ha[pl] * fy};
            const int cs[4] = {c0, c0 + 1, c2, c2 + 1};
#pragma unroll
            for (int e = 0; e < 4; ++e)
              if ((unsigned)cs[e] < (unsigned)kp) ptx::sts16(sArow + a_col(cs[e]), ptx::f32_to_f16(w4[e]));
          }
          if (hb && (unsigned)(ktex - w0) < (unsigned)kp)
            ptx::sts16(sArow + a_col(ktex - w0), (uint16_t)0x3c00u);  // fp16 1.0: + b0
        }
        if (w0 > 0) {  // synchronous staging of an extra window
          fill_table(bb, w0, false);
          ptx::bar_sync(bar_id, 128);
          stage(bb, w0);
        }
        PH(1);
        ptx::cp_async_wait_all();
        ptx::fence_proxy_async_smem();
        ptx::bar_sync(bar_id, 128);
        if (tid < 32) {  // the group's warp 0 issues (one elected lane, warp-uniform code)
          ptx::tc_fence_after();
          // K-step count through a shuffle: a warp-uniform loop (descriptors in uniform
          // registers); measured -0.6 %.  (The same for the hidden layers' weight offset made
          // their 5 dependent MMAs issue back to back: +5.8 %.)
          const int nks = __shfl_sync(0xffffffffu, kpad / 16, 0);
          for (int ks = 0; ks < nks; ++ks) {
            ptx::mma_f16_ss_warp(tmem, a_hi | (a_lo0 + (uint32_t)(ks * 16)), b_hi | (b_lo0 + (uint32_t)(ks * 128)),
                                 idesc_blend, (w0 > 0 || ks > 0) ? 1u : 0u);
          }
          ptx::mma_commit_warp(&sh->mbar[g]);
          if (tid == 0) {  // plain shared-memory counters
            sh->n_tiles[g] += 1u;
            sh->n_kcols[g] += (unsigned)kpad;
          }
        }
        ptx::mbar_wait(&sh->mbar[g], mphase);
        mphase ^= 1u;
      }
      ptx::tc_fence_after();
      PH(2);

      // ---- prefetch chunk c+1 (B tile is free), speculatively for the rays alive now
      const int k1 = k0 + kChunk;
      const bool nxt = GRID ? (k1 / kChunk < kGridKZ && gz0 - (tid >> 5) + (k1 / kChunk) * 4 < P.grid_res)
                            : k1 < P.N;
      if (nxt) prefetch(k1, alive);
      PH(3);

      // ---- MLP layers 1..L-1 on the tensor cores: fp16 activations live in TMEM
      //      (A operand from TMEM), weights in shared memory
      for (int l = 1; l < L; ++l) {
        act_epilogue<ACT>(tmem_row, tmem_row + kTcHD);
        PH(4);
        ptx::tc_fence_before();
        ptx::bar_sync(bar_id, 128);
        if (tid < 32) {
          ptx::tc_fence_after();
          const uint32_t wlo = w_lo0 + (uint32_t)((l - 1) * (kWHidden >> 4));
          const uint32_t id = (l == L - 1) ? idesc_head : idesc_hidden;
          // the head skips its bias K block (4 FADDs at readout instead of an MMA)
          if (l == L - 1) {
            // head: K = 64 as two independent 2-step chains (D and the spare columns
            // [112, 128) of the group's TMEM), summed at readout -- half the dependent steps
#pragma unroll
            for (int ks = 0; ks < 2; ++ks)
#pragma unroll
              for (int hx = 0; hx < 2; ++hx) {
                const int kk = 2 * hx + ks;
                const uint64_t bd = w_hi | (wlo + (uint32_t)(kk * 16));
                ptx::mma_f16_ts_warp(tmem + (hx ? kHeadAlt : 0u), tmem + kTcHD + kk * 8, bd, id, ks > 0 ? 1u : 0u);
              }
          } else {
#pragma unroll
            for (int ks = 0; ks < (int)kWK / 16; ++ks) {
              const uint64_t bd = w_hi | (wlo + (uint32_t)(ks * 16));
              ptx::mma_f16_ts_warp(tmem, tmem + kTcHD + ks * 8, bd, id, ks > 0 ? 1u : 0u);
            }
          }
          ptx::mma_commit_warp(&sh->mbar[g]);
        }
        ptx::mbar_wait(&sh->mbar[g], mphase);
        mphase ^= 1u;
        ptx::tc_fence_after();
        PH(5);
      }
      // ---- head: sigma, rgb (a4)
      uint32_t o4[4];
      ptx::tmem_ld4(tmem_row, o4);
      uint32_t o4b[4];
      ptx::tmem_ld4(tmem_row + kHeadAlt, o4b);
      ptx::tmem_ld_wait();
#pragma unroll
      for (int e = 0; e < 4; ++e) o4[e] = __float_as_uint(__uint_as_float(o4[e]) + __uint_as_float(o4b[e]));
      ptx::tc_fence_before();
      float sigma = 0.0f, c0 = 0.0f, c1 = 0.0f, c2 = 0.0f;
      if (sv) {
        // an inf / NaN anywhere upstream (G or an fp16 activation out of range) reaches the
        // head: count it (range flag bit 1)
        const float chk = __uint_as_float(o4[0]) + __uint_as_float(o4[1]) + __uint_as_float(o4[2]) +
                          __uint_as_float(o4[3]);
        n_range += (fabsf(chk) < INFINITY) ? 0u : 1u;
        const float *bh = sh->head_bias;  // shared memory: broadcast reads
        const float x = __uint_as_float(o4[0]) + bh[0] + P.dshift;
        sigma = __logf(1.0f + __expf(-fabsf(x))) + fmaxf(x, 0.0f);
        const float s = 1.0f + 2.0f * P.weps;
        c0 = __fdividef(s, 1.0f + __expf(-(__uint_as_float(o4[1]) + bh[1]))) - P.weps;
        c1 = __fdividef(s, 1.0f + __expf(-(__uint_as_float(o4[2]) + bh[2]))) - P.weps;
        c2 = __fdividef(s, 1.0f + __expf(-(__uint_as_float(o4[3]) + bh[3]))) - P.weps;
        n_samples++;
      }
      if constexpr (GRID) {
        if (sv) {
          const int64_t n3 = (int64_t)P.grid_res * P.grid_res * P.grid_res;
          const int64_t rg = ((int64_t)gz * P.grid_res + gy) * P.grid_res + gx;
          P.grid_sigma[rg] = sigma;
          if (P.grid_rgb) {
            P.grid_rgb[rg] = c0;
            P.grid_rgb[n3 + rg] = c1;
            P.grid_rgb[2 * n3 + rg] = c2;
          }
        }
        k0 = k1;
        have = nxt;  // uniform over the group: no vote
        continue;
      }
      // ---- a5: composite the ray's 8 samples (8-lane segmented scan)
      const float tau = sv ? sigma * delta : 0.0f;
      float S = tau;
#pragma unroll
      for (int s = 1; s < kChunk; s <<= 1) {
        const float y = __shfl_up_sync(0xffffffffu, S, s, kChunk);
        if (q >= s) S += y;
      }
      const float Tk = T * __expf(-(S - tau));
      const float w = Tk * (1.0f - __expf(-tau));
      acc0 += w * c0;
      acc1 += w * c1;
      acc2 += w * c2;
      const float Stot = __shfl_sync(0xffffffffu, S, kChunk - 1, kChunk);
      T = T * __expf(-Stot);
      if (alive && P.term_eps > 0.0f && T < P.term_eps) {
        if (nxt && q == 0) n_term++;
        alive = false;
      }
      k0 = k1;
      have = nxt && ptx::bar_red_or(bar_id, 128, alive);
      PH(6);
    }
    ptx::cp_async_wait_all();  // a prefetch for a chunk nobody needs may still be landing
    // ---- ray epilogue: reduce the 8 lanes, write rgb/alpha (+ DDIM x_{t-1})
#pragma unroll
    for (int s = kChunk / 2; s > 0; s >>= 1) {
      acc0 += __shfl_xor_sync(0xffffffffu, acc0, s, kChunk);
      acc1 += __shfl_xor_sync(0xffffffffu, acc1, s, kChunk);
      acc2 += __shfl_xor_sync(0xffffffffu, acc2, s, kChunk);
    }
    if (!GRID && pix && q < 3) ray_epilogue(P, v, i, j, q, q == 0 ? acc0 : (q == 1 ? acc1 : acc2), T);
  }

#ifdef DMV3D_PHASES
  if (P.counters && tid == 0)
    for (int i = 0; i < 8; ++i) atomicAdd(P.counters + 8 + i, ph_acc[i]);
#endif
  if (__any_sync(0xffffffffu, n_range != 0u) && (tid & 31) == 0)
    atomicOr(reinterpret_cast<unsigned int *>(const_cast<void *>(P.tp)) + 1, 2u);
  if (P.counters) {
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
      n_range += __shfl_xor_sync(0xffffffffu, n_range, s);
      n_hit += __shfl_xor_sync(0xffffffffu, n_hit, s);
      n_samples += __shfl_xor_sync(0xffffffffu, n_samples, s);
      n_term += __shfl_xor_sync(0xffffffffu, n_term, s);
      n_rays += __shfl_xor_sync(0xffffffffu, n_rays, s);
    }
    if ((tid & 31) == 0) {
      atomicAdd(P.counters + 0, (unsigned long long)n_hit);
      atomicAdd(P.counters + 1, (unsigned long long)n_samples);
      atomicAdd(P.counters + 2, (unsigned long long)n_term);
      atomicAdd(P.counters + 3, (unsigned long long)n_rays);
      if (n_range) atomicAdd(P.counters + 6, (unsigned long long)n_range);
    }
    if (tid == 0) {  // MMA rows issued (128 per blend window) and staged K columns
      atomicAdd(P.counters + 4, 128ull * sh->n_tiles[g]);
      atomicAdd(P.counters + 5, (unsigned long long)sh->n_kcols[g]);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(sh->tmem_base, kTmemCols);
  }
}

// ------------------------------------------------------------------ launch
template <int NG, bool GRID, int ACT>
static cudaError_t launch_k1a(const RenderParams &P, int sms, int64_t npatch, cudaStream_t st) {
  const size_t s1 = tc_smem_bytes<NG>(P.L);
  cudaError_t e = cudaFuncSetAttribute(render_tc_kernel<NG, GRID, ACT>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s1);
  if (e != cudaSuccess) return e;
  int grid = sms;
  if ((int64_t)grid * NG > npatch) grid = (int)((npatch + NG - 1) / NG);
  render_tc_kernel<NG, GRID, ACT><<<grid, 128 * NG, s1, st>>>(P);
  return cudaGetLastError();
}
template <int NG, bool GRID>
static cudaError_t launch_k1(const RenderParams &P, int sms, int64_t npatch, cudaStream_t st) {
  if (P.act == 1) return launch_k1a<NG, GRID, 1>(P, sms, npatch, st);  // SiLU
  if (P.act == 2) return launch_k1a<NG, GRID, 2>(P, sms, npatch, st);  // softplus
  return launch_k1a<NG, GRID, 0>(P, sms, npatch, st);                  // ReLU
}

// K0 alone (shared with the tensor-core backward): G = F W0^T + b0 * bscale (fp16)
// into the workspace, patch counter zeroed.  The bias is split over the three planes
// except for the mean, whose A weights carry the 1/3; the half-pixel mode adds it
// through the bias row instead.
cudaError_t launch_preproject(const RenderParams &P, cudaStream_t st) {
  uint8_t *ws = static_cast<uint8_t *>(P.ws);
  __half *G = reinterpret_cast<__half *>(ws + kWsHeader);
  unsigned int *counter = reinterpret_cast<unsigned int *>(ws);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int ntex = 3 * P.R * P.R;
  const int A = P.V / P.V_asset;  // assets of a batched launch (each its own G block)
  const size_t s0 = (size_t)kTcHD * P.C * 4;
  auto kern = P.tp_fp8 ? preproject_kernel<true> : preproject_kernel<false>;
  // range flags (header word 1) of this call: cleared here, raised by K0 (bit 0) and
  // the render kernel (bit 1)
  cudaError_t e = cudaMemsetAsync(counter + 1, 0, sizeof(unsigned int), st);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s0);
  if (e != cudaSuccess) return e;
  const float bscale = P.smode != 0 ? 0.0f : (P.agg == 0 ? 1.0f : (1.0f / 3.0f));
  const uint8_t *F = static_cast<const uint8_t *>(P.tp);
  const size_t esz = P.tp_fp8 ? 1 : 2;
  const __nv_bfloat16 *W0 = reinterpret_cast<const __nv_bfloat16 *>(P.w[0]);
  const bool cat = P.agg == 2;
  // blocks per SM: 2 for a paper-sized triplane (each block loads W0, 20 KiB, once; 8
  // measured 1 % slower on cfg2), 4 (the register limit) for large / batched triplanes
  auto k0_blocks = [&](int64_t texels) { return texels > (int64_t)64 * 1024 ? 4 : 2; };
  const size_t gs = ((size_t)ntex + 1) * kTcHD;  // G block of one asset
  if (!cat) {  // all assets' texels in one launch
    const int64_t nt = (int64_t)A * ntex;
    int64_t g0 = (nt * 8 + 255) / 256;  // one warp per 4 texels
    if (g0 > (int64_t)sms * k0_blocks(nt)) g0 = (int64_t)sms * k0_blocks(nt);
    kern<<<(int)g0, 256, s0, st>>>(F, (int)nt, P.C, P.C, W0, P.b[0], bscale, P.tp_scale, G, counter,
                                   G + (size_t)ntex * kTcHD, ntex, A, counter + 1);
    return cudaGetLastError();
  }
  // concat: plane p of every asset is projected by its own column block of W0
  const int nt = P.R * P.R;
  int g0 = (nt * 8 + 255) / 256;
  if (g0 > sms * k0_blocks(nt)) g0 = sms * k0_blocks(nt);
  for (int a = 0; a < A; ++a)
    for (int pl = 0; pl < 3; ++pl) {
      const bool first = a == 0 && pl == 0;
      kern<<<g0, 256, s0, st>>>(F + ((size_t)a * 3 + pl) * nt * P.C * esz, nt, P.C, 3 * P.C,
                                W0 + (size_t)pl * P.C, P.b[0], bscale, P.tp_scale,
                                G + a * gs + (size_t)pl * nt * kTcHD, first ? counter : nullptr,
                                first ? G + (size_t)ntex * kTcHD : nullptr, ntex, first ? A : 0,
                                counter + 1);
      e = cudaGetLastError();
      if (e != cudaSuccess) return e;
    }
  return cudaSuccess;
}

// P.grid_res > 0 selects the density-grid mode (row f3)
cudaError_t launch_render_tc(const RenderParams &P0, cudaStream_t st) {
  const bool grid_mode = P0.grid_res > 0;
  if (!grid_mode && P0.ray_end <= P0.ray_begin) return cudaSuccess;
  if (!P0.ws) return cudaErrorInvalidValue;
  RenderParams P = P0;
  uint8_t *ws = static_cast<uint8_t *>(P.ws);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // K0: G = F W0^T + b0 * bscale (fp16), zero the patch counter (a later ray-range launch
  // of the same step reuses G and only resets the counter)
  cudaError_t e = P.reuse_g ? cudaMemsetAsync(ws, 0, sizeof(unsigned int), st) : launch_preproject(P, st);
  if (e != cudaSuccess) return e;
  // K1: persistent render, one CTA per SM; as many groups as shared memory allows
  P.tp = ws;  // the render kernel reads the workspace (counter + G)
  const bool ng4 = tc_smem_bytes<4>(P.L) + sizeof(TcShared<4>) <= kSmemLimit;
  timer_begin(P.timer, st);
  if (grid_mode) {
    const int Gr = P.grid_res;
    const int64_t nb = (int64_t)((Gr + 7) / 8) * ((Gr + 3) / 4) * ((Gr + 4 * kGridKZ - 1) / (4 * kGridKZ));
    e = ng4 ? launch_k1<4, true>(P, sms, nb, st) : launch_k1<2, true>(P, sms, nb, st);
  } else {
    const int64_t HW = (int64_t)P.H * P.W;
    const int v_lo = (int)(P.ray_begin / HW), v_hi = (int)((P.ray_end - 1) / HW);
    int64_t npatch = (int64_t)(v_hi - v_lo + 1) * ((P.H + 3) / 4) * ((P.W + 3) / 4);
    if (P.tile_size > 0) {
      int64_t first = 0, n = 0;
      owned_tiles(v_lo, v_hi, P.H, P.W, P.tile_size, P.tile_rank, P.tile_count, first, n);
      npatch = n * (P.tile_size / 4) * (P.tile_size / 4);
      if (npatch == 0) {
        timer_end(P.timer, st);
        return cudaSuccess;
      }
    }
    e = ng4 ? launch_k1<4, false>(P, sms, npatch, st) : launch_k1<2, false>(P, sms, npatch, st);
  }
  timer_end(P.timer, st);
  return e;
}

}  // namespace dmv3d
