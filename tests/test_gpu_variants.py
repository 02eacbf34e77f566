"""GPU parity of the row-f4 variants against the oracle (-m gpu): half-pixel texel
addressing with zero padding (grid_sample align_corners=False, pinned in
test_oracle_pins) and the concat aggregation (MLP input [f_XY, f_XZ, f_YZ]),
through every stage: texel indices bit-exact, features and decode at the fp32 bar,
full renders on both engines, the density grid and the renderer backward."""
import numpy as np
import pytest
import torch

import oracle
from paper_2605_18052_b200 import api
from paper_2605_18052_b200 import workloads as wl

from helpers import dev_cams, dev_workload, flat_ids, pick

pytestmark = pytest.mark.gpu

FP32_TOL = 1e-5
RGB_TOL, ALPHA_TOL = 2e-2, 1e-2
HP = "halfpixel_zeros"
OAGG = {"mean": oracle.AGG_MEAN, "sum": oracle.AGG_SUM, "concat": oracle.AGG_CONCAT}
OMODE = {"align_corners": 0, HP: 1}


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _cams(H, W):
    return wl.concat_cameras(wl.input_cameras(H, W, 3), wl.novel_cameras(H, W, 2, seed=31))


# ------------------------------------------------------------------ a3 texels
@pytest.mark.parametrize("jitter", [False, True])
def test_halfpixel_texels_bit_exact(jitter):
    """Unclamped lower texel index (-1 .. R-1) and fraction per plane axis equal the
    oracle's bit for bit; N = 160 puts the first/last samples within half a texel of
    the faces, so the zero-padded border cells are exercised."""
    cams = _cams(8, 8)
    intr, c2w = dev_cams(cams)
    R, N = 64, 160
    t_k, pts, texel, frac = api.dmv3d_debug_sample_points(intr, c2w, 8, 8, R, N, jitter=jitter,
                                                          seed=5, sample_mode=HP)
    pts, texel, frac = (x.cpu().numpy() for x in (pts, texel, frac))
    ids = np.arange(cams.num_views * 64)
    o, d, tn, tf, h = oracle.ray_geometry(cams, ids)
    seen = set()
    for r in np.random.default_rng(2).choice(ids[h == 1], 40, replace=False):
        for k in range(N):
            _, p = oracle.sample_point(o[r], d[r], tn[r], tf[r], N, k, int(jitter), 5, int(r))
            assert np.array_equal(pts[r, k].view(np.uint32), p.view(np.uint32))
            for pl, (a, b) in enumerate([(0, 1), (0, 2), (1, 2)]):
                for e, ax in enumerate((a, b)):
                    i0, f = oracle.texel_coord(p[ax], -1, 1, R, sample_mode=1)
                    assert texel[r, k, pl, e] == i0
                    assert frac[r, k, pl, e].view(np.uint32) == np.float32(f).view(np.uint32)
                    seen.add(int(i0))
    assert -1 in seen and R - 1 in seen  # both zero-padded borders reached


# ------------------------------------------------------------------ a3/a4 stages
@pytest.mark.parametrize("C,dtype", [(8, "f32"), (32, "bf16"), (4, "f32")])
@pytest.mark.parametrize("agg", ["mean", "sum", "concat"])
@pytest.mark.parametrize("mode", ["align_corners", HP])
def test_features_variants(C, dtype, agg, mode):
    if agg == "concat" and C == 32:
        C = 16  # concat feature width 3C must be an instantiated SIMT shape (12/24/48/96)
    R = 13
    tp = wl.random_triplane(R, C, seed=C)
    if dtype == "bf16":
        tp = wl.round_to_bf16(tp)
    if dtype == "bf16" and C % 8:
        pytest.skip("bf16 storage needs C % 8 == 0")
    pts = np.random.default_rng(C).uniform(-1.1, 1.1, (901, 3)).astype(np.float32)
    dt = torch.bfloat16 if dtype == "bf16" else torch.float32
    g = api.dmv3d_debug_sample_features(torch.from_numpy(tp).cuda().to(dt), torch.from_numpy(pts).cuda(),
                                        agg, sample_mode=mode).cpu().numpy()
    want = oracle.point_features(tp, pts, OAGG[agg], sample_mode=OMODE[mode])
    assert g.shape == want.shape
    assert np.max(np.abs(g - want)) < 6e-6 * max(1.0, np.abs(want).max())


@pytest.mark.parametrize("C,H,L,agg,mode", [(4, 16, 2, "concat", "align_corners"),
                                            (32, 64, 4, "concat", HP),
                                            (16, 32, 3, "concat", "align_corners"),
                                            (32, 64, 4, "mean", HP)])
def test_decode_variants(C, H, L, agg, mode):
    K = 3 * C if agg == "concat" else C
    tp = wl.blob_triplane(20, C, seed=3)
    m = wl.blob_mlp(K, H, L, seed=4)
    pts = np.random.default_rng(5).uniform(-1, 1, (513, 3)).astype(np.float32)
    g = api.dmv3d_debug_decode(torch.from_numpy(tp).cuda(), api.DeviceMLP.from_host(m, "f32"),
                               torch.from_numpy(pts).cuda(), agg, sample_mode=mode).cpu().numpy()
    want = oracle.decode_points(tp, m, pts, OAGG[agg], sample_mode=OMODE[mode])
    err = np.abs(g - want)
    assert np.max(err[:, 1:]) < FP32_TOL
    assert np.max(err[:, 0] / np.maximum(1.0, want[:, 0])) < 1e-5


# ------------------------------------------------------------------ a1-a6 render
def _workload(C, agg, R=24, H=18, W=14, N=48, L=4, HD=64, dtype="f32", seed=1):
    K = 3 * C if agg == "concat" else C
    tp = wl.blob_triplane(R, C, seed)
    m = wl.blob_mlp(K, HD, L, seed + 1)
    if dtype == "bf16":
        tp, m = wl.round_to_bf16(tp), wl.bf16_mlp(m)
    return wl.Workload("f4", tp, _cams(H, W), m, N, dtype)


def _render(w, agg, mode, engine, ids=None, term_eps=0.0, bg=(1.0, 1.0, 1.0)):
    tp, intr, c2w, mlp = dev_workload(w)
    H, W = w.cameras.height, w.cameras.width
    rgb, alpha = api.dmv3d_render_views(tp, intr, c2w, H, W, mlp, samples_per_ray=w.samples_per_ray,
                                        engine=engine, agg=agg, sample_mode=mode, term_eps=term_eps,
                                        bg=bg)
    rgb, alpha = rgb.cpu().numpy(), alpha.cpu().numpy()
    if ids is None:
        orgb, oalpha = oracle.render_views(w.triplane, w.cameras, w.mlp, w.samples_per_ray,
                                           OAGG[agg], bg=bg, sample_mode=OMODE[mode])
        return rgb, alpha, orgb, oalpha
    orgb, oalpha = oracle.render_rays(w.triplane, w.cameras, w.mlp, w.samples_per_ray, ids,
                                      OAGG[agg], bg=bg, sample_mode=OMODE[mode])
    g_rgb, g_alpha = pick(rgb, alpha, ids, H, W)
    return g_rgb, g_alpha, orgb, oalpha


@pytest.mark.parametrize("C,HD,agg,mode", [(32, 64, "mean", HP), (16, 32, "concat", "align_corners"),
                                           (32, 64, "concat", HP), (8, 16, "sum", HP)])
def test_simt_render_variants(C, HD, agg, mode):
    w = _workload(C, agg, HD=HD)
    rgb, alpha, orgb, oalpha = _render(w, agg, mode, "simt", bg=(0.2, 0.5, 0.9))
    assert np.max(np.abs(rgb - orgb)) < FP32_TOL
    assert np.max(np.abs(alpha - oalpha)) < FP32_TOL
    assert oalpha.max() > 0.5  # the field is not empty


@pytest.mark.parametrize("C,agg,mode,R", [(32, "mean", HP, 64), (32, "concat", "align_corners", 64),
                                          (80, "concat", HP, 64), (24, "sum", HP, 16),
                                          (16, "mean", HP, 128)])
def test_tc_render_variants(C, agg, mode, R):
    """Tensor-core engine: concat projects each plane with its own block of W0; the
    half-pixel mode adds b0 through the extra bias column.  R = 128 forces
    multi-window blends (the bias column may land in a later window)."""
    w = _workload(C, agg, R=R, H=28, W=22, N=64, dtype="bf16")
    rgb, alpha, orgb, oalpha = _render(w, agg, mode, "tcgen05", term_eps=1e-4)
    assert np.max(np.abs(rgb - orgb)) < RGB_TOL
    assert np.max(np.abs(alpha - oalpha)) < ALPHA_TOL
    assert oalpha.max() > 0.5


def test_tc_halfpixel_concat_bench_shape_sampled():
    """cfg-sized image (256^2, C=80, N=128) with both variants, sampled rays."""
    w = _workload(80, "concat", R=64, H=256, W=256, N=128, dtype="bf16", seed=7)
    ids = flat_ids(w.cameras.num_views, 256, 256, 1024, seed=4)
    g_rgb, g_alpha, orgb, oalpha = _render(w, "concat", HP, "tcgen05", ids=ids, term_eps=1e-4)
    assert np.max(np.abs(g_rgb - orgb)) < RGB_TOL
    assert np.max(np.abs(g_alpha - oalpha)) < ALPHA_TOL


# ------------------------------------------------------------------ f3 / f1 with the variants
@pytest.mark.parametrize("engine,dtype", [("simt", "f32"), ("tcgen05", "bf16")])
@pytest.mark.parametrize("agg,mode", [("concat", HP), ("mean", HP)])
def test_density_grid_variants(engine, dtype, agg, mode):
    C = 32
    K = 3 * C if agg == "concat" else C
    tp = wl.blob_triplane(12, C, seed=4)
    m = wl.blob_mlp(K, 64, 4, seed=5)
    if dtype == "bf16":
        tp, m = wl.round_to_bf16(tp), wl.bf16_mlp(m)
    dt = torch.bfloat16 if dtype == "bf16" else torch.float32
    G = 21
    sigma, rgb = api.dmv3d_density_grid(torch.from_numpy(tp).cuda().to(dt),
                                        api.DeviceMLP.from_host(m, dtype), G, agg=agg, engine=engine,
                                        sample_mode=mode)
    osig, orgb = oracle.density_grid(tp, m, G, OAGG[agg], sample_mode=OMODE[mode])
    tol = FP32_TOL if engine == "simt" else RGB_TOL
    s = sigma.cpu().numpy()
    assert np.all(s > 0)
    assert np.max(np.abs(s - osig) / np.maximum(1.0, osig)) < tol
    assert np.max(np.abs(rgb.cpu().numpy() - orgb)) < tol


def _close(g, o, rel=1e-4):
    g, o = np.asarray(g, np.float64), np.asarray(o, np.float64)
    return np.max(np.abs(g - o)) <= rel * max(np.max(np.abs(o)), 1e-30) + 1e-7


@pytest.mark.parametrize("C,HD,agg,mode", [(8, 16, "concat", HP), (16, 32, "concat", "align_corners"),
                                           (32, 64, "mean", HP)])
def test_backward_variants(C, HD, agg, mode):
    K = 3 * C if agg == "concat" else C
    tp = wl.blob_triplane(12, C, seed=7, kappa=4.0)
    m = wl.blob_mlp(K, HD, 3, seed=8)
    cams = wl.concat_cameras(wl.input_cameras(10, 9, 2), wl.novel_cameras(10, 9, 1, seed=9))
    w = wl.Workload("bw", tp, cams, m, 40, "f32")
    t, intr, c2w, mlp = dev_workload(w)
    rng = np.random.default_rng(C)
    g = rng.normal(size=(3, 3, 10, 9)).astype(np.float32)
    gA = rng.normal(size=(3, 10, 9)).astype(np.float32)
    dF, dW, db = api.dmv3d_render_backward(t, intr, c2w, 10, 9, mlp, torch.from_numpy(g).cuda(),
                                           torch.from_numpy(gA).cuda(), samples_per_ray=40,
                                           agg=agg, sample_mode=mode, bg=(0.3, 0.5, 0.7))
    oF, oW, ob = oracle.render_backward(tp, cams, m, 40, g, gA, agg=OAGG[agg], bg=(0.3, 0.5, 0.7),
                                        sample_mode=OMODE[mode])
    assert np.max(np.abs(oF)) > 0
    assert _close(dF.cpu().numpy(), oF)
    for l in range(3):
        assert _close(dW[l].cpu().numpy(), oW[l]), l
        assert _close(db[l].cpu().numpy(), ob[l]), l


# ------------------------------------------------------------------ fp8 triplane storage
def _fp8_setup(scale, C=32, H=12, W=11, N=48):
    tp = wl.blob_triplane(16, C, seed=2)
    codes, vals = wl.to_e4m3(tp, scale)
    m = wl.bf16_mlp(wl.blob_mlp(C, 64, 4, seed=3))
    cams = _cams(H, W)
    dev = torch.device("cuda")
    t8 = torch.from_numpy(codes).to(dev).view(torch.float8_e4m3fn)
    intr, c2w = dev_cams(cams)
    return vals, m, cams, t8, intr, c2w, api.DeviceMLP.from_host(m, "bf16", dev)


@pytest.mark.parametrize("scale", [1.0, 0.375])
def test_fp8_triplane_render_tc(scale):
    """Row f4: E4M3 triplane storage (value = scale * e4m3) on the tensor-core engine
    equals the oracle rendering the dequantised values, at the bf16 TC bar."""
    vals, m, cams, t8, intr, c2w, mlp = _fp8_setup(scale)
    H, W = cams.height, cams.width
    rgb, alpha = api.dmv3d_render_views(t8, intr, c2w, H, W, mlp, samples_per_ray=48,
                                        engine="tcgen05", fp8_scale=scale)
    orgb, oalpha = oracle.render_views(vals, cams, m, 48)
    assert np.max(np.abs(rgb.cpu().numpy() - orgb)) < RGB_TOL
    assert np.max(np.abs(alpha.cpu().numpy() - oalpha)) < ALPHA_TOL


def test_fp8_triplane_backward_tc():
    vals, m, cams, t8, intr, c2w, mlp = _fp8_setup(0.5)
    H, W = cams.height, cams.width
    rng = np.random.default_rng(5)
    g = rng.normal(size=(cams.num_views, 3, H, W)).astype(np.float32)
    dF, dW, db = api.dmv3d_render_backward(t8, intr, c2w, H, W, mlp, torch.from_numpy(g).cuda(),
                                           samples_per_ray=48, engine="tcgen05", fp8_scale=0.5)
    oF, oW, ob = oracle.render_backward(vals, cams, m, 48, g)
    rel = lambda a, b: np.max(np.abs(a - b)) / np.max(np.abs(b))  # noqa: E731
    assert rel(dF.cpu().numpy(), oF) < 2e-2
    for l in range(4):
        assert rel(dW[l].cpu().numpy(), oW[l]) < 2e-2 and rel(db[l].cpu().numpy(), ob[l]) < 2e-2


def test_fp8_triplane_needs_tc_engine():
    _, _, cams, t8, intr, c2w, mlp = _fp8_setup(1.0)
    with pytest.raises(api._abi.DMV3DError) as e:
        api.dmv3d_render_views(t8, intr, c2w, cams.height, cams.width, mlp, samples_per_ray=8,
                               engine="simt")
    assert e.value.status == 2  # UNSUPPORTED


def test_fp8_triplane_density_grid_tc():
    vals, m, cams, t8, intr, c2w, mlp = _fp8_setup(0.75)
    G = 19
    sigma, rgb = api.dmv3d_density_grid(t8, mlp, G, engine="tcgen05", fp8_scale=0.75)
    osig, orgb = oracle.density_grid(vals, m, G)
    s = sigma.cpu().numpy()
    assert np.max(np.abs(s - osig) / np.maximum(1.0, osig)) < RGB_TOL
    assert np.max(np.abs(rgb.cpu().numpy() - orgb)) < RGB_TOL
