"""Pins for the CPU oracle (-m "not gpu").

Each test checks the oracle against something other than itself: a closed
form from the paper's definitions, an invariant, a special case that reduces
to a library routine (torch grid_sample / linear / softplus), or brute force.
Citations: PAPER.md line numbers; SURVEY.md §8c C3 pin ids (P1..P13).
"""
import math

import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle
from paper_2605_18052_b200 import workloads as wl


# ----------------------------------------------------------------------------- helpers
def const_field_mlp(in_dim, sigma=None, rgb_bias=0.0, hidden=16):
    """MLP whose output ignores the features: sigma = softplus(shift), c = sigmoid(rgb_bias)."""
    w0 = np.zeros((hidden, in_dim), np.float32)
    b0 = np.zeros(hidden, np.float32)
    w1 = np.zeros((4, hidden), np.float32)
    b1 = np.array([0.0, rgb_bias, rgb_bias, rgb_bias], np.float32)
    shift = math.log(math.expm1(sigma)) if sigma is not None else 0.0
    return wl.MLP([w0, w1], [b0, b1], 0, shift, 0.0)


def torch_features(tp, pts, agg=oracle.AGG_MEAN):
    """Library special case: bilinear align-corners lookup == grid_sample(align_corners=True)
    on each plane with the plane's two world axes as (x=column, y=row) (readings A2, A3)."""
    t = torch.from_numpy(tp.astype(np.float64))  # [3][R][R][C]
    p = torch.from_numpy(pts.astype(np.float64))
    out = 0
    for pl, (a, b) in enumerate([(0, 1), (0, 2), (1, 2)]):
        img = t[pl].permute(2, 0, 1)[None]  # [1][C][R(row)][R(col)]
        grid = torch.stack([p[:, a], p[:, b]], -1)[None, None]  # x -> col, y -> row
        out = out + F.grid_sample(img, grid, mode="bilinear", padding_mode="border",
                                  align_corners=True)[0, :, 0, :].T
    if agg == oracle.AGG_MEAN:
        out = out / 3.0
    return out.numpy()


def torch_mlp(m, h0):
    h = torch.from_numpy(np.atleast_2d(h0).astype(np.float64))
    L = m.num_layers
    for l in range(L):
        h = F.linear(h, torch.from_numpy(m.weights[l].astype(np.float64)),
                     torch.from_numpy(m.biases[l].astype(np.float64)))
        if l < L - 1:
            h = {0: F.relu, 1: F.silu, 2: lambda x: F.softplus(x, threshold=1e9)}[m.hidden_act](h)
    sigma = F.softplus(h[:, 0] + m.density_shift, threshold=1e9)
    rgb = torch.sigmoid(h[:, 1:]) * (1 + 2 * m.rgb_widen_eps) - m.rgb_widen_eps
    return torch.cat([sigma[:, None], rgb], 1).numpy()


# ----------------------------------------------------------------------------- schedule (P10)
def test_schedule_golden_values(golden):
    g = golden["schedule_cosine"]
    ab = oracle.cosine_alpha_bar(g["T"], g["s"])
    for t, v in g["alpha_bar"].items():
        assert abs(ab[int(t)] - v) < g["tol"], (t, ab[int(t)], v)


def test_schedule_telescopes_and_decreases():
    """prod_{j<=t}(1-beta_j) telescopes to f(t+1)/f(0) while the clip is inactive;
    alpha_bar is strictly decreasing."""
    T, s = 1000, 0.008
    ab = oracle.cosine_alpha_bar(T, s)
    f = lambda t: math.cos(((t / T) + s) / (1 + s) * math.pi / 2) ** 2
    for t in range(0, 990):
        assert abs(ab[t] - f(t + 1) / f(0)) < 1e-12 * max(1.0, 1.0 / ab[t]) + 1e-15
    assert np.all(np.diff(ab) < 0)
    assert 0 < ab[-1] < ab[0] <= 1


# ----------------------------------------------------------------------------- ray generation (a1)
def test_rays_project_back_to_their_pixels():
    """Independent inverse: o + t d, mapped world->camera with the inverse of c2w and
    projected with the pinhole intrinsics, lands on the pixel centre (j+1/2, i+1/2)."""
    cams = wl.concat_cameras(wl.input_cameras(12, 10, 4), wl.novel_cameras(12, 10, 3, seed=7))
    rng = np.random.default_rng(0)
    ids = rng.integers(0, cams.num_views * 120, 200)
    o, d, tn, tf, hit = oracle.ray_geometry(cams, ids)
    for q, r in enumerate(ids):
        v, rem = divmod(int(r), 120)
        i, j = divmod(rem, 10)
        M = cams.c2w[v].astype(np.float64)
        assert np.all(o[q] == cams.c2w[v][:, 3])
        assert abs(np.linalg.norm(d[q].astype(np.float64)) - 1) < 1e-6
        X = o[q].astype(np.float64) + 3.0 * d[q].astype(np.float64)
        xc = M[:, :3].T @ (X - M[:, 3])
        fx, fy, cx, cy = cams.intrinsics[v].astype(np.float64)
        assert xc[2] > 0
        assert abs(fx * xc[0] / xc[2] + cx - (j + 0.5)) < 1e-4
        assert abs(fy * xc[1] / xc[2] + cy - (i + 0.5)) < 1e-4


def test_axis_ray_p7():
    """Odd image, camera at (2.7,0,0): the centre pixel ray is exactly -x, and its
    chord through [-1,1]^3 is [r-1, r+1]."""
    cams = wl.axis_camera(15, 15)
    r = 7 * 15 + 7
    o, d, tn, tf, hit = oracle.ray_geometry(cams, [r])
    assert hit[0] == 1
    assert np.all(d[0] == np.array([-1, 0, 0], np.float32))
    assert o[0][0] == np.float32(2.7)
    assert abs(tn[0] - 1.7) <= 2.4e-7 and abs(tf[0] - 3.7) <= 4.8e-7


def test_slab_brute_force():
    """hit == some point of the ray (t>=0) is strictly inside the box, by dense
    fp64 marching; for hits, the entry/exit points lie on the box surface."""
    cams = wl.concat_cameras(wl.input_cameras(16, 16, 4),
                             wl.concat_cameras(wl.novel_cameras(16, 16, 4, seed=11),
                                               wl.away_camera(16, 16)))
    ids = np.arange(cams.num_views * 256)
    o, d, tn, tf, hit = oracle.ray_geometry(cams, ids)
    ts = np.linspace(0, 6, 6001)
    for q in range(len(ids)):
        P = o[q][None].astype(np.float64) + ts[:, None] * d[q][None].astype(np.float64)
        inside = np.all(np.abs(P) < 1 - 1e-4, axis=1).any()
        near_in = np.all(np.abs(P) <= 1 + 1e-4, axis=1).any()
        if inside:
            assert hit[q] == 1
        if not near_in:
            assert hit[q] == 0
        if hit[q]:
            pe = o[q].astype(np.float64) + float(tn[q]) * d[q]
            px = o[q].astype(np.float64) + float(tf[q]) * d[q]
            if tn[q] > 0:
                assert abs(np.max(np.abs(pe)) - 1) < 1e-5
            assert abs(np.max(np.abs(px)) - 1) < 1e-5
        else:
            assert tn[q] == 0 and tf[q] == 0


def test_away_camera_all_miss_p5(golden):
    cams = wl.away_camera(8, 8)
    tp = wl.random_triplane(8, 4, 3)
    m = wl.random_mlp(4, 16, 2, 3)
    rgb, alpha = oracle.render_views(tp, cams, m, 16, bg=(0.2, 0.4, 0.6))
    assert np.all(alpha == 0.0)
    for c, b in enumerate((0.2, 0.4, 0.6)):
        assert np.all(rgb[:, c] == b)


# ----------------------------------------------------------------------------- samples (a2)
def test_samples_midpoints_partition_the_chord():
    o = np.array([2.7, 0.3, -0.2], np.float32)
    d = np.array([-1, 0.05, 0.02], np.float32)
    d = (d / np.linalg.norm(d)).astype(np.float32)
    tn, tf, N = np.float32(1.75), np.float32(3.5), 64
    ts = np.array([oracle.sample_point(o, d, tn, tf, N, k)[0] for k in range(N)], np.float64)
    delta = (float(tf) - float(tn)) / N
    assert np.all(np.diff(ts) > 0)
    assert abs(ts[0] - (tn + delta / 2)) < 1e-6 and abs(ts[-1] - (tf - delta / 2)) < 1e-6
    assert np.max(np.abs(np.diff(ts) - delta)) < 1e-6
    assert abs(ts.mean() - (float(tn) + float(tf)) / 2) < 1e-6


def test_jitter_is_uniform_and_stratified():
    u = np.array([oracle.jitter(1234, s) for s in range(20000)])
    assert u.min() >= 0 and u.max() < 1
    assert abs(u.mean() - 0.5) < 0.01 and abs(u.var() - 1 / 12) < 0.005
    assert np.all(u * 2**24 == np.floor(u * 2**24))  # 24-bit grid
    o = np.zeros(3, np.float32)
    d = np.array([1, 0, 0], np.float32)
    ts = [oracle.sample_point(o, d, 0.0, 1.0, 8, k, 1, 99, 5)[0] for k in range(8)]
    for k, t in enumerate(ts):
        assert k / 8 <= t < (k + 1) / 8  # one sample per stratum


# ----------------------------------------------------------------------------- texels + gather (a3)
def test_texel_centres_align_corners():
    R = 9
    for idx in range(R):
        q = -1.0 + 2.0 * idx / (R - 1)
        i0, f = oracle.texel_coord(q, -1.0, 1.0, R)
        if idx < R - 1:
            assert (i0, f) == (idx, 0.0)
        else:
            assert (i0, f) == (R - 2, 1.0)
    assert oracle.texel_coord(-1.5, -1, 1, R) == (0, 0.0)  # clamped
    assert oracle.texel_coord(1.5, -1, 1, R) == (R - 2, 1.0)


def test_linear_plane_reproduced_exactly_p4():
    """F = a*col + b*row + e  =>  bilinear sample = a*px + b*py + e; points
    on a dyadic grid so px is exact in fp32 and the identity holds to fp64 rounding."""
    R, C = 9, 5
    tp, a, b, e = wl.linear_triplane(R, C, seed=4)
    rng = np.random.default_rng(1)
    pts = (-1.0 + rng.integers(0, 129, (300, 3)) / 64.0).astype(np.float32)
    feats = oracle.point_features(tp, pts, oracle.AGG_SUM)
    want = np.zeros_like(feats)
    for pl, (ax, bx) in enumerate([(0, 1), (0, 2), (1, 2)]):
        px = (pts[:, ax].astype(np.float64) + 1) * 4
        py = (pts[:, bx].astype(np.float64) + 1) * 4
        want += a[pl][None] * px[:, None] + b[pl][None] * py[:, None] + e[pl][None]
    # the plane values themselves are fp32-rounded: compare with tolerance on that scale
    tpf = tp.astype(np.float64)
    exact = np.zeros_like(feats)
    for pl, (ax, bx) in enumerate([(0, 1), (0, 2), (1, 2)]):
        px = (pts[:, ax].astype(np.float64) + 1) * 4
        py = (pts[:, bx].astype(np.float64) + 1) * 4
        ix = np.minimum(np.floor(px).astype(int), R - 2)
        iy = np.minimum(np.floor(py).astype(int), R - 2)
        fx, fy = px - ix, py - iy
        # the fp32 plane is linear within each cell up to its own rounding
        exact += ((1 - fx) * (1 - fy))[:, None] * tpf[pl, iy, ix] + (fx * (1 - fy))[:, None] * tpf[pl, iy, ix + 1] \
            + ((1 - fx) * fy)[:, None] * tpf[pl, iy + 1, ix] + (fx * fy)[:, None] * tpf[pl, iy + 1, ix + 1]
    assert np.max(np.abs(feats - want)) < 1e-5  # fp32 storage of the linear field
    assert np.max(np.abs(feats - exact)) < 1e-12


def test_features_match_grid_sample():
    """Library special case: mean of three grid_sample(align_corners=True) lookups.
    Catches swapped planes/axes, transposed rows/cols and wrong corner weights."""
    R, C = 12, 7
    tp = wl.random_triplane(R, C, seed=5)
    rng = np.random.default_rng(2)
    pts = rng.uniform(-1, 1, (500, 3)).astype(np.float32)
    got = oracle.point_features(tp, pts, oracle.AGG_MEAN)
    want = torch_features(tp, pts, oracle.AGG_MEAN)
    assert np.max(np.abs(got - want)) < 2e-6
    got_s = oracle.point_features(tp, pts, oracle.AGG_SUM)
    assert np.max(np.abs(got_s - 3 * got)) < 1e-12


# ----------------------------------------------------------------------------- MLP (a4)
@pytest.mark.parametrize("act", [0, 1, 2])
def test_mlp_matches_torch(act):
    m = wl.random_mlp(10, 16, 4, seed=3)
    m.hidden_act, m.density_shift, m.rgb_widen_eps = act, -1.0, 0.001
    h0 = np.random.default_rng(3).normal(0, 2, (64, 10))
    got = oracle.mlp_decode(m, h0)
    want = torch_mlp(m, h0)
    assert np.max(np.abs(got - want)) < 1e-12


def test_blob_mlp_density_closed_form():
    """Benchmark MLP: sigma = softplus(20*max(h0[0],0) - 6)."""
    m = wl.blob_mlp(80, 64, 4)
    h0 = np.random.default_rng(4).normal(0, 3, (50, 80))
    got = oracle.mlp_decode(m, h0)[:, 0]
    x = 20 * np.maximum(h0[:, 0], 0) - 6
    want = np.log1p(np.exp(-np.abs(x))) + np.maximum(x, 0)
    assert np.max(np.abs(got - want)) < 1e-9


# ----------------------------------------------------------------------------- compositing (a5)
def _axis_case(half, sigma, rgb_bias, N, bg=(1.0, 1.0, 1.0)):
    cams = wl.axis_camera(15, 15)
    r = 7 * 15 + 7
    tp = wl.const_triplane(4, 4, 0.3)
    m = const_field_mlp(4, sigma, rgb_bias)
    rgb, alpha = oracle.render_rays(tp, cams, m, N, [r], bg=bg, aabb_min=(-half,) * 3,
                                    aabb_max=(half,) * 3)
    o, d, tn, tf, hit = oracle.ray_geometry(cams, [r], (-half,) * 3, (half,) * 3)
    delta = float(np.float32(np.float32(tf[0] - tn[0]) / np.float32(N)))
    return rgb[0], alpha[0], delta


def test_beer_lambert_p1(golden):
    g = golden["beer_lambert"]
    for N in (1, 7, 64, 128):
        rgb, alpha, delta = _axis_case(g["chord"] / 2, g["sigma"], 0.0, N)
        assert abs(alpha - (1 - math.exp(-g["sigma"] * N * delta))) < 1e-12  # exact in N*delta
        assert abs(alpha - g["alpha"]) < g["tol"] + 2 * 3e-7  # chord = 1.5 up to fp32 geometry
    # T_64 of a 128-sample ray = transmittance after half the chord = 1 - alpha(N=64, half chord)
    rgb, alpha64, _ = _axis_case(g["chord"] / 4, g["sigma"], 0.0, 64)
    assert abs((1 - alpha64) - g["T_64_of_128"]) < g["tol"] + 3e-7


def test_constant_colour_p2(golden):
    g = golden["constant_colour"]
    bias = np.float32(math.log(g["c"] / (1 - g["c"])))
    c = 1 / (1 + math.exp(-float(bias)))
    for N in (3, 128):
        rgb, alpha, delta = _axis_case(g["chord"] / 2, g["sigma"], bias, N, bg=(g["bg"],) * 3)
        A = 1 - math.exp(-g["sigma"] * N * delta)
        assert np.max(np.abs(rgb - (c * A + g["bg"] * (1 - A)))) < 1e-12
        assert np.max(np.abs(rgb - g["rgb"])) < g["tol"] + 1e-6
        # bg = 0: colour times opacity
        rgb0, alpha0, _ = _axis_case(g["chord"] / 2, g["sigma"], bias, N, bg=(0.0,) * 3)
        assert np.max(np.abs(rgb0 - c * alpha0)) < 1e-12


def test_weights_sum_and_bg_linearity_p3():
    """rgb(bg) - rgb(0) = bg * T_N = bg * (1 - A); 0 <= A <= 1; rgb in the convex hull."""
    w = wl.make_workload("cfg1")
    tp = wl.random_triplane(8, 4, 9)
    m = wl.random_mlp(4, 16, 2, 9)
    m.density_shift = 1.0
    cams = w.cameras
    rgb1, a1 = oracle.render_views(tp, cams, m, 16, bg=(0.3, 0.6, 0.9))
    rgb0, a0 = oracle.render_views(tp, cams, m, 16, bg=(0.0, 0.0, 0.0))
    assert np.all(a1 == a0)
    assert np.all((a0 >= 0) & (a0 <= 1))
    for c, b in enumerate((0.3, 0.6, 0.9)):
        assert np.max(np.abs(rgb1[:, c] - rgb0[:, c] - b * (1 - a0))) < 1e-12
    assert np.all(rgb0 >= 0) and np.all(rgb0 <= a0[:, None] + 1e-15)


def test_render_brute_force_p6():
    """cfg1: the oracle render equals an independent per-sample evaluation: torch
    grid_sample + torch MLP at the sample points, composited with the closed form
    w_k = exp(-sum_{j<k} tau_j) (1 - exp(-tau_k))."""
    w = wl.make_workload("cfg1")
    V, H, W = w.cameras.num_views, w.cameras.height, w.cameras.width
    rgb, alpha = oracle.render_views(w.triplane, w.cameras, w.mlp, w.samples_per_ray)
    ids = np.arange(V * H * W)
    o, d, tn, tf, hit = oracle.ray_geometry(w.cameras, ids)
    N = w.samples_per_ray
    assert hit.mean() > 0.5
    for r in ids:
        v, pix = divmod(int(r), H * W)
        i, j = divmod(pix, W)
        got = np.array([rgb[v, 0, i, j], rgb[v, 1, i, j], rgb[v, 2, i, j], alpha[v, i, j]])
        if not hit[r]:
            assert np.all(got == np.array([1, 1, 1, 0]))
            continue
        pts = np.stack([oracle.sample_point(o[r], d[r], tn[r], tf[r], N, k)[1] for k in range(N)])
        dec = torch_mlp(w.mlp, torch_features(w.triplane, pts))
        delta = float(np.float32(np.float32(tf[r] - tn[r]) / np.float32(N)))
        tau = dec[:, 0] * delta
        excl = np.concatenate([[0.0], np.cumsum(tau)[:-1]])
        wk = np.exp(-excl) * (1 - np.exp(-tau))
        A = 1 - np.exp(-tau.sum())
        want = np.concatenate([(wk[:, None] * dec[:, 1:]).sum(0) + (1 - A), [A]])
        assert np.max(np.abs(got - want)) < 1e-5, r


def test_blob_workload_opacity_mix():
    """Workload check: the blob field has both opaque and clear rays."""
    w = wl.make_workload("cfg2")
    rng = np.random.default_rng(0)
    ids = rng.choice(w.num_rays, 300, replace=False)
    rgb, alpha = oracle.render_rays(w.triplane, w.cameras, w.mlp, w.samples_per_ray, ids)
    o, d, tn, tf, hit = oracle.ray_geometry(w.cameras, ids)
    a = alpha[hit == 1]
    assert (a > 0.99).mean() > 0.25 and (a < 0.01).mean() > 0.25


# ----------------------------------------------------------------------------- DDIM (a6)
def test_ddim_consistency_p8(golden):
    g = golden["ddim_consistency"]
    ab = oracle.cosine_alpha_bar()
    x0 = np.full((1, 3, 2, 2), g["x0"])
    eps = np.full_like(x0, g["eps"])
    x_t = math.sqrt(ab[g["t"]]) * x0 + math.sqrt(1 - ab[g["t"]]) * eps
    rgb = (x0 + 1) / 2  # x0 = 2 rgb - 1 (reading A15)
    out = oracle.ddim_step(ab, g["t"], g["t_prev"], x_t, rgb)
    want = math.sqrt(ab[g["t_prev"]]) * x0 + math.sqrt(1 - ab[g["t_prev"]]) * eps
    assert np.max(np.abs(out - want)) < 1e-12
    assert np.max(np.abs(out - g["x_prev"])) < g["tol"]


def test_ddim_final_step_and_keep_mask_p9():
    ab = oracle.cosine_alpha_bar()
    rng = np.random.default_rng(5)
    x_t = rng.normal(size=(3, 3, 4, 5))
    rgb = rng.uniform(size=(3, 3, 4, 5))
    z = rng.normal(size=(3, 3, 4, 5))
    out = oracle.ddim_step(ab, 0, -1, x_t, rgb, z, eta=1.0)
    assert np.max(np.abs(out - (2 * rgb - 1))) < 1e-12  # fully denoised
    out = oracle.ddim_step(ab, 980, 960, x_t, rgb, z, eta=0.5, keep_mask=[1, 0, 0])
    assert np.all(out[0] == x_t[0])  # conditioning view kept noise-free
    assert not np.allclose(out[1], x_t[1])


def test_ddim_eta1_is_ddpm_posterior_p9(golden):
    """eta=1: the deterministic part equals the DDPM posterior mean
    mu = sqrt(ab_p) b/(1-ab_t) x0 + sqrt(a)(1-ab_p)/(1-ab_t) x_t with a = ab_t/ab_p,
    b = 1-a, and the noise scale is sqrt(beta_tilde) = sqrt((1-ab_p)/(1-ab_t) b)."""
    g = golden["ddim_eta1_sigma"]
    ab = oracle.cosine_alpha_bar()
    for t, tp_ in ((980, 960), (500, 480), (40, 20)):
        abt, abp = ab[t], ab[tp_]
        a = abt / abp
        b = 1 - a
        rng = np.random.default_rng(t)
        x_t = rng.normal(size=(1, 3, 3, 3))
        rgb = rng.uniform(size=(1, 3, 3, 3))
        x0 = 2 * rgb - 1
        mean = oracle.ddim_step(ab, t, tp_, x_t, rgb, np.zeros_like(x_t), eta=1.0)
        mu = math.sqrt(abp) * b / (1 - abt) * x0 + math.sqrt(a) * (1 - abp) / (1 - abt) * x_t
        assert np.max(np.abs(mean - mu)) < 1e-10
        one = oracle.ddim_step(ab, t, tp_, x_t, rgb, np.ones_like(x_t), eta=1.0)
        sig = float(np.mean(one - mean))
        assert abs(sig - math.sqrt((1 - abp) / (1 - abt) * b)) < 1e-10
        if t == g["t"]:
            assert abs(sig - g["sigma_t"]) < g["tol"]


# ----------------------------------------------------------------------------- f2 Plucker rays
def test_plucker_closed_forms():
    """r = (o x d, d): the moment is orthogonal to d, equals p x d for any
    point p on the ray (fp64 recompute), and vanishes for a ray through the origin."""
    cams = wl.concat_cameras(wl.input_cameras(7, 9, 4), wl.novel_cameras(7, 9, 3, seed=8))
    ids = np.arange(cams.num_views * 63)
    pl = oracle.plucker(cams, ids).astype(np.float64)
    o, d, *_ = oracle.ray_geometry(cams, ids)
    m, dd = pl[:, :3], pl[:, 3:]
    assert np.array_equal(dd, d.astype(np.float64))
    assert np.max(np.abs(np.sum(m * dd, 1))) < 1e-5
    for t in (0.7, 2.3):
        p = o.astype(np.float64) + t * d.astype(np.float64)
        assert np.max(np.abs(np.cross(p, d.astype(np.float64)) - m)) < 2e-6
    ax = oracle.plucker(wl.axis_camera(15, 15), [7 * 15 + 7])[0]
    assert np.all(ax[:3] == 0) and np.array_equal(ax[3:], np.array([-1, 0, 0], np.float32))


# ----------------------------------------------------------------------------- f3 density grid
def test_density_grid_on_texel_lattice():
    """With G = R the grid points sit exactly on the texel lattice (align-corners), so
    no interpolation happens: the density grid equals the torch MLP applied to the mean
    of the three texels each point projects to (row f3)."""
    R, C = 9, 8
    tp = wl.random_triplane(R, C, seed=6)
    m = wl.random_mlp(C, 16, 3, seed=6)
    sigma, rgb = oracle.density_grid(tp, m, R)
    pts = oracle.grid_points(R)
    assert np.array_equal(pts[:R, 0], np.linspace(-1, 1, R).astype(np.float32))  # x fastest
    assert np.all(pts[R * R * R - 1] == 1.0) and np.all(pts[0] == -1.0)
    idx = np.stack(np.meshgrid(np.arange(R), np.arange(R), np.arange(R), indexing="ij"), -1)
    iz, iy, ix = idx[..., 0].ravel(), idx[..., 1].ravel(), idx[..., 2].ravel()
    t64 = tp.astype(np.float64)
    h0 = (t64[0, iy, ix] + t64[1, iz, ix] + t64[2, iz, iy]) / 3.0
    want = torch_mlp(m, h0)
    assert np.max(np.abs(sigma.ravel() - want[:, 0])) < 1e-12
    assert np.max(np.abs(rgb.reshape(3, -1).T - want[:, 1:])) < 1e-12


# ----------------------------------------------------------------------------- f4 variants
def test_halfpixel_zero_padding_matches_grid_sample():
    """Row f4: half-pixel texel centres with zero padding are exactly
    grid_sample(align_corners=False, padding_mode='zeros') on each plane."""
    R, C = 7, 5
    tp = wl.random_triplane(R, C, seed=11)
    pts = np.random.default_rng(11).uniform(-1, 1, (400, 3)).astype(np.float32)
    got = oracle.point_features(tp, pts, oracle.AGG_SUM, sample_mode=oracle.SAMPLE_HALFPIXEL_ZEROS)
    t = torch.from_numpy(tp.astype(np.float64))
    p = torch.from_numpy(pts.astype(np.float64))
    want = 0
    for pl, (a, b) in enumerate([(0, 1), (0, 2), (1, 2)]):
        img = t[pl].permute(2, 0, 1)[None]
        grid = torch.stack([p[:, a], p[:, b]], -1)[None, None]
        want = want + F.grid_sample(img, grid, mode="bilinear", padding_mode="zeros",
                                    align_corners=False)[0, :, 0, :].T
    # fp32 fractions (reading A3): |df| <= ~R*2^-24 per axis, x texel deltas, x3 planes summed
    assert np.max(np.abs(got - want.numpy())) < 6e-6
    # near the faces the half-pixel mode fades to zero, unlike align-corners
    i0, f = oracle.texel_coord(-1.0, -1.0, 1.0, R, sample_mode=1)
    assert (i0, f) == (-1, 0.5)


def test_concat_aggregation_stacks_the_planes():
    """Row f4: concat aggregation (A4 alternative) = [f_XY, f_XZ, f_YZ], each the
    align-corners bilinear lookup of its plane; the mean is their average."""
    R, C = 9, 4
    tp = wl.random_triplane(R, C, seed=12)
    pts = np.random.default_rng(12).uniform(-1, 1, (300, 3)).astype(np.float32)
    cat = oracle.point_features(tp, pts, oracle.AGG_CONCAT)
    assert cat.shape == (300, 3 * C)
    mean = torch_features(tp, pts, oracle.AGG_MEAN)
    assert np.max(np.abs((cat[:, :C] + cat[:, C:2 * C] + cat[:, 2 * C:]) / 3 - mean)) < 2e-6
    single = torch_features(np.stack([tp[1], tp[1], tp[1]]), pts, oracle.AGG_SUM)  # not the XZ axes
    assert np.max(np.abs(cat[:, C:2 * C] - single / 3)) > 1e-3  # planes are not interchangeable


# ----------------------------------------------------------------------------- f4 in-kernel noise
def test_in_kernel_noise_is_standard_normal():
    """Row f4: the counter-based DDIM noise is N(0,1): Kolmogorov-Smirnov distance to
    the normal CDF, moments, and no lag-1 correlation (z enters x_{t-1} = ... + sigma_t z,
    PAPER.md:1102 'isotropic Gaussian')."""
    from scipy import stats
    z = oracle.noise(2024, 60000)
    assert stats.kstest(z, "norm").statistic < 0.008
    assert abs(z.mean()) < 0.02 and abs(z.var() - 1) < 0.03
    assert abs(np.corrcoef(z[:-1], z[1:])[0, 1]) < 0.02
    assert not np.array_equal(oracle.noise(1, 100), oracle.noise(2, 100))


# ----------------------------------------------------------------------------- f1 backward
@pytest.mark.parametrize("act,agg,mode", [(2, oracle.AGG_MEAN, 0), (1, oracle.AGG_SUM, 0),
                                          (0, oracle.AGG_MEAN, 0), (2, oracle.AGG_CONCAT, 1)])
def test_render_backward_matches_central_differences(act, agg, mode):
    """Row f1 ("differentiable volume rendering"): the oracle's analytic
    gradients equal central finite differences of the oracle's own forward render,
    (L(x+h) - L(x-h)) / 2h with h = 1e-6 on fp64 inputs (SPEC.md:112 methodology)."""
    rng = np.random.default_rng(act)
    tp = rng.normal(0, 0.8, (3, 5, 5, 4))
    m = wl.random_mlp(12 if agg == oracle.AGG_CONCAT else 4, 8, 3, seed=act)
    m = wl.MLP([w.astype(np.float64) for w in m.weights], [b.astype(np.float64) for b in m.biases],
               act, 0.3, 0.01)
    cams = wl.input_cameras(4, 4, 2)
    N = 7
    g = rng.normal(size=(2, 3, 4, 4))
    gA = rng.normal(size=(2, 4, 4))

    def loss(tp_, m_):
        rgb, alpha = oracle.render_views(tp_, cams, m_, N, agg=agg, bg=(0.3, 0.6, 0.9), threads=1,
                                         sample_mode=mode)
        return float(np.sum(g * rgb) + np.sum(gA * alpha))

    dF, dW, db = oracle.render_backward(tp, cams, m, N, g, gA, agg=agg, bg=(0.3, 0.6, 0.9),
                                        sample_mode=mode)
    h = 1e-6
    flat = np.argsort(-np.abs(dF).ravel())[:12]  # entries the rays actually touch
    flat = np.concatenate([flat, rng.choice(dF.size, 6, replace=False)])
    for f in flat:
        e = np.zeros(dF.size)
        e[f] = h
        fd = (loss(tp + e.reshape(tp.shape), m) - loss(tp - e.reshape(tp.shape), m)) / (2 * h)
        assert abs(fd - dF.ravel()[f]) < 1e-6 * max(1.0, abs(fd)), (f, fd, dF.ravel()[f])
    for l in range(m.num_layers):
        for which in ("w", "b"):
            arr = m.weights[l] if which == "w" else m.biases[l]
            grad = dW[l] if which == "w" else db[l]
            for f in rng.choice(arr.size, min(5, arr.size), replace=False):
                def with_delta(dv):
                    a2 = arr.copy().ravel()
                    a2[f] += dv
                    ws = [x.copy() for x in m.weights]
                    bs = [x.copy() for x in m.biases]
                    (ws if which == "w" else bs)[l] = a2.reshape(arr.shape)
                    return wl.MLP(ws, bs, act, 0.3, 0.01)
                fd = (loss(tp, with_delta(h)) - loss(tp, with_delta(-h))) / (2 * h)
                assert abs(fd - grad.ravel()[f]) < 1e-6 * max(1.0, abs(fd)), (l, which, f)
