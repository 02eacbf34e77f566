"""GPU parity: libdmv3d (through the C ABI) vs the CPU oracle on the same seeded
inputs (-m gpu).  Bars: bit-exact ray/sample
geometry and indices; fp32 engine max-abs 1e-5 on rgb/alpha; bf16
tensor-core engine 2e-2 rgb / 1e-2 alpha; x_{t-1} by the DDIM Lipschitz
bound of the rgb tolerance."""
import numpy as np
import pytest
import torch

import oracle
from paper_2605_18052_b200 import api, schedule
from paper_2605_18052_b200 import workloads as wl

from helpers import ddim_tol, dev_cams, dev_workload, flat_ids, pick

pytestmark = pytest.mark.gpu

FP32_TOL = 1e-5


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.init()


def _mixed_cams(H=9, W=11):
    return wl.concat_cameras(wl.concat_cameras(wl.input_cameras(H, W, 4), wl.novel_cameras(H, W, 3, seed=21)),
                             wl.away_camera(H, W))


# ------------------------------------------------------------------ a1/a2 geometry
def test_ray_geometry_bit_exact():
    cams = wl.concat_cameras(_mixed_cams(), wl.axis_camera(9, 11))
    intr, c2w = dev_cams(cams)
    o_d, tn_tf, hit = api.dmv3d_debug_ray_geometry(intr, c2w, 9, 11)
    torch.cuda.synchronize()
    ids = np.arange(cams.num_views * 99)
    o, d, tn, tf, h = oracle.ray_geometry(cams, ids)
    g = o_d.cpu().numpy()
    assert np.array_equal(g[:, :3].view(np.uint32), o.view(np.uint32))
    assert np.array_equal(g[:, 3:].view(np.uint32), d.view(np.uint32))
    gt = tn_tf.cpu().numpy()
    assert np.array_equal(gt[:, 0].view(np.uint32), tn.view(np.uint32))
    assert np.array_equal(gt[:, 1].view(np.uint32), tf.view(np.uint32))
    assert np.array_equal(hit.cpu().numpy().astype(np.int32), h)
    assert 0 < h.mean() < 1


def test_ray_geometry_shard_and_box():
    cams = _mixed_cams(16, 16)
    intr, c2w = dev_cams(cams)
    lo, hi = (-0.6, -0.8, -0.7), (0.9, 0.5, 0.75)
    o_d, tn_tf, hit = api.dmv3d_debug_ray_geometry(intr, c2w, 16, 16, lo, hi, ray_range=(300, 1700))
    ids = np.arange(300, 1700)
    o, d, tn, tf, h = oracle.ray_geometry(cams, ids, lo, hi)
    gt = tn_tf.cpu().numpy()
    assert np.array_equal(gt[:, 0].view(np.uint32), tn.view(np.uint32))
    assert np.array_equal(gt[:, 1].view(np.uint32), tf.view(np.uint32))
    assert np.array_equal(hit.cpu().numpy().astype(np.int32), h)


@pytest.mark.parametrize("jitter", [False, True])
def test_sample_points_and_texels_bit_exact(jitter):
    cams = _mixed_cams(8, 8)
    intr, c2w = dev_cams(cams)
    R, N = 64, 37
    t_k, pts, texel, frac = api.dmv3d_debug_sample_points(intr, c2w, 8, 8, R, N, jitter=jitter,
                                                          seed=77)
    t_k, pts, texel, frac = (x.cpu().numpy() for x in (t_k, pts, texel, frac))
    ids = np.arange(cams.num_views * 64)
    o, d, tn, tf, h = oracle.ray_geometry(cams, ids)
    rng = np.random.default_rng(1)
    for r in rng.choice(ids[h == 1], 60, replace=False):
        for k in range(N):
            t, p = oracle.sample_point(o[r], d[r], tn[r], tf[r], N, k, int(jitter), 77, int(r))
            assert t_k[r, k].view(np.uint32) == np.float32(t).view(np.uint32)
            assert np.array_equal(pts[r, k].view(np.uint32), p.view(np.uint32))
            for pl, (a, b) in enumerate([(0, 1), (0, 2), (1, 2)]):
                ia, fa = oracle.texel_coord(p[a], -1, 1, R)
                ib, fb = oracle.texel_coord(p[b], -1, 1, R)
                assert tuple(texel[r, k, pl]) == (ia, ib)
                assert frac[r, k, pl, 0].view(np.uint32) == np.float32(fa).view(np.uint32)
                assert frac[r, k, pl, 1].view(np.uint32) == np.float32(fb).view(np.uint32)
    miss = ids[h == 0]
    assert np.all(t_k[miss] == 0) and np.all(texel[miss] == 0)


# ------------------------------------------------------------------ a3/a4 stages
@pytest.mark.parametrize("C,dtype", [(4, "f32"), (32, "f32"), (80, "f32"), (32, "bf16"), (80, "bf16")])
def test_features_match_oracle(C, dtype):
    R = 17
    tp = wl.random_triplane(R, C, seed=C)
    if dtype == "bf16":
        tp = wl.round_to_bf16(tp)
    rng = np.random.default_rng(C)
    pts = rng.uniform(-1.1, 1.1, (777, 3)).astype(np.float32)
    dt = torch.bfloat16 if dtype == "bf16" else torch.float32
    g = api.dmv3d_debug_sample_features(torch.from_numpy(tp).cuda().to(dt),
                                        torch.from_numpy(pts).cuda()).cpu().numpy()
    want = oracle.point_features(tp, pts)
    assert np.max(np.abs(g - want)) < 2e-6 * max(1.0, np.abs(want).max())
    gs = api.dmv3d_debug_sample_features(torch.from_numpy(tp).cuda().to(dt),
                                         torch.from_numpy(pts).cuda(), "sum").cpu().numpy()
    assert np.max(np.abs(gs - 3 * want)) < 6e-6 * max(1.0, np.abs(want).max())


@pytest.mark.parametrize("C,H,L,act", [(4, 16, 2, 0), (32, 64, 4, 0), (80, 64, 4, 0), (80, 64, 3, 1),
                                       (16, 32, 5, 2)])
def test_decode_matches_oracle(C, H, L, act):
    tp = wl.blob_triplane(20, C, seed=3)
    m = wl.blob_mlp(C, H, L, seed=4)
    m.hidden_act, m.density_shift, m.rgb_widen_eps = act, -0.5, 0.002
    pts = np.random.default_rng(5).uniform(-1, 1, (513, 3)).astype(np.float32)
    g = api.dmv3d_debug_decode(torch.from_numpy(tp).cuda(), api.DeviceMLP.from_host(m, "f32"),
                               torch.from_numpy(pts).cuda()).cpu().numpy()
    want = oracle.decode_points(tp, m, pts)
    err = np.abs(g - want)
    assert np.max(err[:, 1:]) < FP32_TOL
    assert np.max(err[:, 0] / np.maximum(1.0, want[:, 0])) < 1e-5  # ~K*eps_f32 over 3 layers


# ------------------------------------------------------------------ a1-a5 render
def _render_both(w, term_eps=0.0, engine="simt", bg=(1.0, 1.0, 1.0), ids=None, **kw):
    tp, intr, c2w, mlp = dev_workload(w)
    H, W = w.cameras.height, w.cameras.width
    rgb, alpha = api.dmv3d_render_views(tp, intr, c2w, H, W, mlp, samples_per_ray=w.samples_per_ray,
                                        term_eps=term_eps, engine=engine, bg=bg, **kw)
    rgb, alpha = rgb.cpu().numpy(), alpha.cpu().numpy()
    if ids is None:
        orgb, oalpha = oracle.render_views(w.triplane, w.cameras, w.mlp, w.samples_per_ray, bg=bg)
        return rgb, alpha, orgb, oalpha
    orgb, oalpha = oracle.render_rays(w.triplane, w.cameras, w.mlp, w.samples_per_ray, ids, bg=bg)
    g_rgb, g_alpha = pick(rgb, alpha, ids, H, W)
    return g_rgb, g_alpha, orgb, oalpha


@pytest.mark.parametrize("term_eps", [0.0, 1e-6])
def test_render_cfg1_full_image(term_eps):
    w = wl.make_workload("cfg1")
    rgb, alpha, orgb, oalpha = _render_both(w, term_eps)
    assert np.max(np.abs(rgb - orgb)) < FP32_TOL
    assert np.max(np.abs(alpha - oalpha)) < FP32_TOL


def _mid_workload(dtype="f32", C=32, N=40, H=24, W=20, L=4):
    tp = wl.blob_triplane(16, C, seed=12)
    m = wl.blob_mlp(C, 64, L, seed=13)
    if dtype == "bf16":
        tp, m = wl.round_to_bf16(tp), wl.bf16_mlp(m)
    cams = wl.concat_cameras(wl.input_cameras(H, W, 2), wl.novel_cameras(H, W, 1, seed=14))
    return wl.Workload("mid", tp, cams, m, N, dtype)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_render_ragged_full_image_simt(dtype):
    """Ragged image (24x20), ragged chunk (N=40 = 32 + 8), several views; the SIMT
    engine computes in fp32, so bf16 storage is held to the fp32 bar."""
    w = _mid_workload(dtype)
    rgb, alpha, orgb, oalpha = _render_both(w, 1e-6, bg=(0.2, 0.5, 0.9))
    assert np.max(np.abs(rgb - orgb)) < FP32_TOL
    assert np.max(np.abs(alpha - oalpha)) < FP32_TOL


def test_render_cfg2_fp32_sampled():
    w = wl.make_workload("cfg2")
    ids = flat_ids(4, 128, 128, 768, seed=2)
    g_rgb, g_alpha, orgb, oalpha = _render_both(w, 1e-6, ids=ids)
    assert np.max(np.abs(g_rgb - orgb)) < FP32_TOL
    assert np.max(np.abs(g_alpha - oalpha)) < FP32_TOL


def test_render_edge_cases():
    # all rays miss -> background, alpha 0 (exactly)
    w = _mid_workload()
    w.cameras = wl.away_camera(8, 8)
    rgb, alpha, orgb, oalpha = _render_both(w, bg=(0.25, 0.5, 0.75))
    assert np.all(alpha == 0) and np.all(rgb[:, 0] == 0.25) and np.all(rgb[:, 2] == 0.75)
    # one sample per ray, 1x1 image
    w = _mid_workload(N=1, H=1, W=1)
    rgb, alpha, orgb, oalpha = _render_both(w)
    assert np.max(np.abs(rgb - orgb)) < FP32_TOL and np.max(np.abs(alpha - oalpha)) < FP32_TOL
    # tiny triplane (R = 2)
    w = _mid_workload(C=8, N=33, H=5, W=7, L=2)
    w.triplane = wl.random_triplane(2, 8, 3)
    w.mlp = wl.random_mlp(8, 16, 2, 3)
    rgb, alpha, orgb, oalpha = _render_both(w)
    assert np.max(np.abs(rgb - orgb)) < FP32_TOL and np.max(np.abs(alpha - oalpha)) < FP32_TOL


def test_termination_bound_and_counters():
    w = _mid_workload()
    tp, intr, c2w, mlp = dev_workload(w)
    H, W = w.cameras.height, w.cameras.width
    cnt0 = torch.zeros(8, dtype=torch.int64, device="cuda")
    cnt1 = torch.zeros(8, dtype=torch.int64, device="cuda")
    full, afull = api.dmv3d_render_views(tp, intr, c2w, H, W, mlp, samples_per_ray=w.samples_per_ray,
                                         term_eps=0.0, counters=cnt0)
    eps = 1e-3
    term, aterm = api.dmv3d_render_views(tp, intr, c2w, H, W, mlp, samples_per_ray=w.samples_per_ray,
                                         term_eps=eps, counters=cnt1)
    assert (full - term).abs().max().item() <= eps * 1.01  # reading A14 bound
    assert (afull - aterm).abs().max().item() <= eps * 1.01
    c0, c1 = cnt0.cpu().numpy(), cnt1.cpu().numpy()
    nrays = w.num_rays
    _, _, _, _, hit = oracle.ray_geometry(w.cameras, np.arange(nrays))
    assert c0[3] == nrays and c0[0] == hit.sum() and c0[2] == 0
    assert c0[1] == hit.sum() * w.samples_per_ray
    assert c1[2] > 0 and c1[1] < c0[1]


def test_render_deterministic_and_shard_invariant():
    w = _mid_workload("bf16")
    tp, intr, c2w, mlp = dev_workload(w)
    H, W, N = w.cameras.height, w.cameras.width, w.samples_per_ray
    a, aa = api.dmv3d_render_views(tp, intr, c2w, H, W, mlp, samples_per_ray=N, term_eps=1e-4)
    b, bb = api.dmv3d_render_views(tp, intr, c2w, H, W, mlp, samples_per_ray=N, term_eps=1e-4)
    assert torch.equal(a, b) and torch.equal(aa, bb)  # pin P13
    c = torch.full_like(a, -7.0)
    cc = torch.full_like(aa, -7.0)
    cuts = [0, 101, 777, 1200, w.num_rays]
    for lo, hi in zip(cuts[:-1], cuts[1:]):
        api.dmv3d_render_views(tp, intr, c2w, H, W, mlp, rgb=c, alpha=cc, samples_per_ray=N,
                               term_eps=1e-4, ray_range=(lo, hi))
    assert torch.equal(a, c) and torch.equal(aa, cc)  # pin P12


# ------------------------------------------------------------------ a6 DDIM
@pytest.mark.parametrize("t,t_prev,eta,keep", [(980, 960, 0.0, None), (980, 960, 1.0, [1, 0, 0]),
                                               (500, 480, 0.3, [0, 1, 0]), (20, 0, 1.0, None),
                                               (0, -1, 0.0, None)])
def test_ddim_step_matches_oracle(t, t_prev, eta, keep):
    ab = schedule.cosine_alpha_bar()
    V, H, W = 3, 7, 9  # 3*H*W = 189: not a multiple of 4 -> scalar path
    for (HH, WW) in ((H, W), (8, 8)):
        x_t = wl.gaussian((V, 3, HH, WW), 4)
        rgb = np.random.default_rng(6).uniform(0, 1, (V, 3, HH, WW)).astype(np.float32)
        z = wl.gaussian((V, 3, HH, WW), 5)
        g = api.dmv3d_ddim_step(ab, t, t_prev, torch.from_numpy(x_t).cuda(), torch.from_numpy(rgb).cuda(),
                                torch.from_numpy(z).cuda() if eta > 0 else None, eta,
                                keep).cpu().numpy()
        want = oracle.ddim_step(oracle.cosine_alpha_bar(), t, t_prev, x_t, rgb,
                                z if eta > 0 else None, eta, keep)
        assert np.max(np.abs(g - want)) < 1e-5
        if keep is not None:
            for v, k in enumerate(keep):
                if k:
                    assert np.array_equal(g[v], x_t[v])


@pytest.mark.parametrize("eta,keep", [(0.0, None), (1.0, [1, 0])])
def test_fused_render_ddim_step(eta, keep):
    w = _mid_workload(N=48)
    tp, intr, c2w, mlp = dev_workload(w)
    H, W = w.cameras.height, w.cameras.width
    dv = 2
    ab = schedule.cosine_alpha_bar()
    x_t = wl.gaussian((dv, 3, H, W), 4)
    z = wl.gaussian((dv, 3, H, W), 5)
    xp, rgb, alpha = api.dmv3d_render_ddim_step(tp, intr, c2w, H, W, mlp, ab, 980, 960,
                                                torch.from_numpy(x_t).cuda(),
                                                torch.from_numpy(z).cuda() if eta else None,
                                                eta, keep, samples_per_ray=w.samples_per_ray,
                                                term_eps=1e-6)
    orgb, oalpha = oracle.render_views(w.triplane, w.cameras, w.mlp, w.samples_per_ray)
    assert np.max(np.abs(rgb.cpu().numpy() - orgb)) < FP32_TOL
    assert np.max(np.abs(alpha.cpu().numpy() - oalpha)) < FP32_TOL
    want = oracle.ddim_step(oracle.cosine_alpha_bar(), 980, 960, x_t, orgb[:dv], z if eta else None,
                            eta, keep)
    assert np.max(np.abs(xp.cpu().numpy() - want)) < ddim_tol(ab, 980, 960, FP32_TOL)


def test_host_buffer_entry_matches_device_entry():
    w = _mid_workload("bf16", N=48)
    tp, intr, c2w, mlp = dev_workload(w)
    H, W = w.cameras.height, w.cameras.width
    ab = schedule.cosine_alpha_bar()
    x_t = torch.from_numpy(wl.gaussian((2, 3, H, W), 4))
    xp, rgb, alpha = api.dmv3d_render_ddim_step(tp, intr, c2w, H, W, mlp, ab, 500, 480, x_t.cuda(),
                                                samples_per_ray=48, term_eps=1e-4)
    ws = api.Workspace()
    hmlp = api.DeviceMLP([x.cpu() for x in mlp.weights], [x.cpu() for x in mlp.biases], "bf16")
    h_xp = torch.empty_like(x_t).pin_memory()
    h_rgb = torch.empty(rgb.shape).pin_memory()
    h_alpha = torch.empty(alpha.shape).pin_memory()
    api.dmv3d_render_ddim_step_host(ws, tp.cpu().pin_memory(), intr.cpu().pin_memory(),
                                    c2w.cpu().pin_memory(), H, W, hmlp, ab, 500, 480,
                                    x_t.pin_memory(), h_xp, h_rgb, h_alpha, samples_per_ray=48,
                                    term_eps=1e-4)
    torch.cuda.synchronize()
    assert torch.equal(h_xp, xp.cpu()) and torch.equal(h_rgb, rgb.cpu())
    assert torch.equal(h_alpha, alpha.cpu())
    ws.close()
