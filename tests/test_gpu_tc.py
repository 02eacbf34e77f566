"""GPU parity of the tensor-core engine (tcgen05/TMEM) against the CPU oracle.

Bar (BASELINE.json north_star): max |rgb - oracle| <= 2e-2, max |alpha - oracle|
<= 1e-2 for the bf16 tensor-core path; x_{t-1} within the DDIM Lipschitz bound
of the rgb bar.  Inputs are bf16 (the oracle reads their exact fp32 upcast)."""
import numpy as np
import pytest
import torch

import oracle
from paper_2605_18052_b200 import api, schedule
from paper_2605_18052_b200 import workloads as wl

from helpers import ddim_tol, dev_workload, flat_ids, pick

pytestmark = pytest.mark.gpu

RGB_TOL, ALPHA_TOL = 2e-2, 1e-2


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _wl(C=80, L=4, R=64, H=48, W=40, N=128, views_in=2, views_novel=1, seed=1, blob=True):
    tp = wl.blob_triplane(R, C, seed) if blob else wl.random_triplane(R, C, seed, 0.7)
    m = wl.blob_mlp(C, 64, L, seed + 1) if blob else wl.random_mlp(C, 64, L, seed + 1)
    tp, m = wl.round_to_bf16(tp), wl.bf16_mlp(m)
    cams = wl.concat_cameras(wl.input_cameras(H, W, views_in),
                             wl.novel_cameras(H, W, views_novel, seed=seed + 2))
    return wl.Workload("tc", tp, cams, m, N, "bf16")


def _tc_render(w, term_eps=1e-4, ids=None, bg=(1.0, 1.0, 1.0), agg="mean", **kw):
    tp, intr, c2w, mlp = dev_workload(w)
    H, W = w.cameras.height, w.cameras.width
    cnt = torch.zeros(8, dtype=torch.int64, device="cuda")
    rgb, alpha = api.dmv3d_render_views(tp, intr, c2w, H, W, mlp, samples_per_ray=w.samples_per_ray,
                                        term_eps=term_eps, engine="tcgen05", bg=bg, agg=agg,
                                        counters=cnt, **kw)
    rgb, alpha = rgb.cpu().numpy(), alpha.cpu().numpy()
    oagg = oracle.AGG_MEAN if agg == "mean" else oracle.AGG_SUM
    if ids is None:
        orgb, oalpha = oracle.render_views(w.triplane, w.cameras, w.mlp, w.samples_per_ray, oagg,
                                           bg=bg, **({"jitter": 1, "seed": kw["seed"]} if kw.get("jitter") else {}))
        return rgb, alpha, orgb, oalpha, cnt.cpu().numpy()
    orgb, oalpha = oracle.render_rays(w.triplane, w.cameras, w.mlp, w.samples_per_ray, ids, oagg,
                                      bg=bg)
    g_rgb, g_alpha = pick(rgb, alpha, ids, H, W)
    return g_rgb, g_alpha, orgb, oalpha, cnt.cpu().numpy()


def _report(rgb, alpha, orgb, oalpha):
    e_rgb, e_a = np.abs(rgb - orgb), np.abs(alpha - oalpha)
    print(f"max|rgb|={e_rgb.max():.3g} mean={e_rgb.mean():.3g}  max|alpha|={e_a.max():.3g} "
          f"mean={e_a.mean():.3g}")
    return e_rgb.max(), e_a.max()


@pytest.mark.parametrize("C,L", [(80, 4), (32, 4), (80, 2), (16, 3)])
def test_tc_render_full_image(C, L):
    w = _wl(C=C, L=L)
    rgb, alpha, orgb, oalpha, cnt = _tc_render(w)
    er, ea = _report(rgb, alpha, orgb, oalpha)
    assert er < RGB_TOL and ea < ALPHA_TOL
    assert cnt[3] == w.num_rays


def test_tc_render_ragged_random_field():
    """Random (non-blob) field, ragged 30x22 image (partial 4x4 patches), N=45
    (partial 8-sample chunk), sum aggregation, coloured background, no termination."""
    w = _wl(C=24, L=4, R=16, H=30, W=22, N=45, blob=False)
    rgb, alpha, orgb, oalpha, _ = _tc_render(w, term_eps=0.0, bg=(0.1, 0.6, 0.3), agg="sum")
    er, ea = _report(rgb, alpha, orgb, oalpha)
    assert er < RGB_TOL and ea < ALPHA_TOL


def test_tc_render_multipass_k():
    """R=128 doubles the texel footprint so some tiles exceed the 128-column MMA
    window and take several accumulate passes."""
    w = _wl(C=16, L=3, R=128, H=32, W=32, N=64)
    rgb, alpha, orgb, oalpha, _ = _tc_render(w)
    er, ea = _report(rgb, alpha, orgb, oalpha)
    assert er < RGB_TOL and ea < ALPHA_TOL


def test_tc_render_jitter():
    w = _wl(C=32, L=4, H=20, W=20, N=64)
    rgb, alpha, orgb, oalpha, _ = _tc_render(w, jitter=True, seed=1234)
    er, ea = _report(rgb, alpha, orgb, oalpha)
    assert er < RGB_TOL and ea < ALPHA_TOL


@pytest.mark.parametrize("lo,hi", [((-0.6, -0.8, -0.7), (0.9, 0.5, 0.75)),   # extents not 2^k
                                   ((-1.0, -1.0, -1.0), (1.0, 3.0, 1.0))])    # 2^k, off-centre
def test_tc_render_box(lo, hi):
    """Other bounding boxes: extents that are not powers of two take the kernel's general
    texel-coordinate path (IEEE division), power-of-two extents its multiply fast path."""
    w = _wl(C=32, L=4, H=24, W=20, N=64)
    tp, intr, c2w, mlp = dev_workload(w)
    rgb, alpha = api.dmv3d_render_views(tp, intr, c2w, 24, 20, mlp, samples_per_ray=64, term_eps=1e-4,
                                        engine="tcgen05", aabb_min=lo, aabb_max=hi)
    orgb, oalpha = oracle.render_views(w.triplane, w.cameras, w.mlp, 64, oracle.AGG_MEAN,
                                       aabb_min=lo, aabb_max=hi)
    er, ea = _report(rgb.cpu().numpy(), alpha.cpu().numpy(), orgb, oalpha)
    assert er < RGB_TOL and ea < ALPHA_TOL
    assert 0.0 < float(alpha.mean()) < 1.0


def test_tc_cfg3_sampled():
    """The benchmark configuration itself (8 views 256^2, C=80, N=128), sampled."""
    w = wl.make_workload("cfg3")
    ids = flat_ids(8, 256, 256, 2048, seed=3)
    g_rgb, g_alpha, orgb, oalpha, cnt = _tc_render(w, ids=ids)
    er, ea = _report(g_rgb, g_alpha, orgb, oalpha)
    assert er < RGB_TOL and ea < ALPHA_TOL
    assert cnt[3] == w.num_rays and cnt[0] > 0.9 * w.num_rays


def test_tc_matches_simt_closely():
    """Both engines on the same bf16 inputs: the tensor-core result stays within the
    bf16 bar of the fp32 SIMT engine everywhere (not only at sampled pixels)."""
    w = _wl(C=80, L=4, H=64, W=64, N=96)
    tp, intr, c2w, mlp = dev_workload(w)
    a = api.dmv3d_render_views(tp, intr, c2w, 64, 64, mlp, samples_per_ray=96, term_eps=1e-4,
                               engine="tcgen05")
    b = api.dmv3d_render_views(tp, intr, c2w, 64, 64, mlp, samples_per_ray=96, term_eps=1e-4,
                               engine="simt")
    assert (a[0] - b[0]).abs().max().item() < RGB_TOL
    assert (a[1] - b[1]).abs().max().item() < ALPHA_TOL


def test_tc_deterministic_and_shard_invariant():
    w = _wl(C=32, L=4, H=24, W=28, N=40)
    tp, intr, c2w, mlp = dev_workload(w)
    H, W = 24, 28
    kw = dict(samples_per_ray=40, term_eps=1e-4, engine="tcgen05")
    a, aa = api.dmv3d_render_views(tp, intr, c2w, H, W, mlp, **kw)
    b, bb = api.dmv3d_render_views(tp, intr, c2w, H, W, mlp, **kw)
    assert torch.equal(a, b) and torch.equal(aa, bb)
    # shards on 4x4-patch boundaries (whole views, whole patch rows): bitwise equal (P12)
    c = torch.full_like(a, -7.0)
    cc = torch.full_like(aa, -7.0)
    cuts = [0, 8 * W, H * W, H * W + 12 * W, w.num_rays]
    for lo, hi in zip(cuts[:-1], cuts[1:]):
        api.dmv3d_render_views(tp, intr, c2w, H, W, mlp, rgb=c, alpha=cc, ray_range=(lo, hi), **kw)
    assert torch.equal(a, c) and torch.equal(aa, cc)
    # cuts through patches change a tile's texel window (the MMA's K order): fp32 rounding only
    c.fill_(-7.0)
    cc.fill_(-7.0)
    cuts = [0, 500, H * W, H * W + 333, w.num_rays]
    for lo, hi in zip(cuts[:-1], cuts[1:]):
        api.dmv3d_render_views(tp, intr, c2w, H, W, mlp, rgb=c, alpha=cc, ray_range=(lo, hi), **kw)
    assert (a - c).abs().max().item() < 1e-6 and (aa - cc).abs().max().item() < 1e-6


@pytest.mark.parametrize("t,t_prev,eta,keep", [(980, 960, 0.0, None), (500, 480, 1.0, [1, 0]),
                                               (0, -1, 0.0, None)])
def test_tc_fused_ddim(t, t_prev, eta, keep):
    w = _wl(C=80, L=4, H=32, W=32, N=64)
    tp, intr, c2w, mlp = dev_workload(w)
    ab = schedule.cosine_alpha_bar()
    x_t = wl.gaussian((2, 3, 32, 32), 4)
    z = wl.gaussian((2, 3, 32, 32), 5)
    xp, rgb, alpha = api.dmv3d_render_ddim_step(tp, intr, c2w, 32, 32, mlp, ab, t, t_prev,
                                                torch.from_numpy(x_t).cuda(),
                                                torch.from_numpy(z).cuda() if eta else None, eta,
                                                keep, samples_per_ray=64, term_eps=1e-4,
                                                engine="tcgen05")
    orgb, oalpha = oracle.render_views(w.triplane, w.cameras, w.mlp, 64)
    er, ea = _report(rgb.cpu().numpy(), alpha.cpu().numpy(), orgb, oalpha)
    assert er < RGB_TOL and ea < ALPHA_TOL
    want = oracle.ddim_step(oracle.cosine_alpha_bar(), t, t_prev, x_t, orgb[:2], z if eta else None,
                            eta, keep)
    assert np.max(np.abs(xp.cpu().numpy() - want)) < ddim_tol(ab, t, t_prev, RGB_TOL)
    if keep:
        assert np.array_equal(xp.cpu().numpy()[0], x_t[0])


def test_tc_all_miss_and_tiny():
    w = _wl(C=16, L=2, H=9, W=9, N=8)
    w.cameras = wl.away_camera(9, 9)
    rgb, alpha, orgb, oalpha, cnt = _tc_render(w, bg=(0.3, 0.2, 0.1))
    assert np.all(alpha == 0) and np.all(rgb[:, 0] == np.float32(0.3))
    assert cnt[0] == 0 and cnt[1] == 0
    w = _wl(C=16, L=2, H=1, W=1, N=1, views_in=1, views_novel=1)
    rgb, alpha, orgb, oalpha, _ = _tc_render(w)
    er, ea = _report(rgb, alpha, orgb, oalpha)
    assert er < RGB_TOL and ea < ALPHA_TOL


@pytest.mark.parametrize("R,C,L,N", [(2, 8, 3, 5), (5, 256, 4, 24), (512, 8, 2, 40)])
def test_tc_extreme_shapes(R, C, L, N):
    """Smallest triplane (R = 2: one cell), the widest supported channel count (C = 256:
    32 KiB of W0 in the pre-projection's shared memory), and R = 512 (texel windows far
    beyond one 128-column MMA pass); odd N (partial chunks)."""
    w = _wl(C=C, L=L, R=R, H=13, W=11, N=N, blob=False)
    rgb, alpha, orgb, oalpha, _ = _tc_render(w, term_eps=0.0)
    er, ea = _report(rgb, alpha, orgb, oalpha)
    assert er < RGB_TOL and ea < ALPHA_TOL


def test_tc_ray_range_shards_cover_the_image():
    """Disjoint ray ranges (cut anywhere, including through 4x4 patches and views) write
    exactly their pixels; together they equal the full render within the TC bar."""
    w = _wl(C=32, L=4, H=14, W=18, N=32)
    tp, intr, c2w, mlp = dev_workload(w)
    H, W = 14, 18
    V = w.cameras.num_views
    full = api.dmv3d_render_views(tp, intr, c2w, H, W, mlp, samples_per_ray=32, engine="tcgen05")
    rgb = torch.full((V, 3, H, W), -7.0, device="cuda")
    alpha = torch.full((V, H, W), -7.0, device="cuda")
    cuts = [0, 37, 252, 253, 400, V * H * W]
    for a, b in zip(cuts[:-1], cuts[1:]):
        api.dmv3d_render_views(tp, intr, c2w, H, W, mlp, rgb=rgb, alpha=alpha, samples_per_ray=32,
                               engine="tcgen05", ray_range=(a, b))
    assert (alpha >= 0).all()  # every pixel written exactly by its shard
    assert (rgb - full[0]).abs().max().item() < 1e-5
    assert (alpha - full[1]).abs().max().item() < 1e-5
