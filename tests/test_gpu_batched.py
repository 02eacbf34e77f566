"""Batched assets (cfg4: 8 assets per GPU) and the fused step's
render-skipping options, on the GPU.

* dmv3d_render_ddim_step_batched renders A assets (own triplane, own cameras,
  shared MLP) in one launch: asset by asset it must be BITWISE equal to the
  single-asset call (same patches, same per-ray op order), and each asset within
  the engine's bar of the CPU oracle.
* want_rgb = want_alpha = False renders only the DDIM views; skip_kept_views
  leaves the kept conditioning view unrendered with x_{t-1} = x_t.
"""
import numpy as np
import pytest
import torch

import oracle
from paper_2605_18052_b200 import api, schedule
from paper_2605_18052_b200 import workloads as wl

from helpers import ddim_tol

pytestmark = pytest.mark.gpu

AB = schedule.cosine_alpha_bar()


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _assets(A, R=16, C=32, H=20, W=24, dv=2, nv=1, dtype="bf16", hp=False):
    tps, cams = [], []
    for a in range(A):
        tp = wl.blob_triplane(R, C, seed=100 + a)
        tps.append(wl.round_to_bf16(tp) if dtype == "bf16" else tp)
        cams.append(wl.concat_cameras(wl.input_cameras(H, W, dv),
                                      wl.novel_cameras(H, W, nv, seed=3 + a)))
    m = wl.blob_mlp(C, 64, 4, seed=2)
    if dtype == "bf16":
        m = wl.bf16_mlp(m)
    x_t = np.stack([wl.gaussian((dv, 3, H, W), 4 + a) for a in range(A)]).astype(np.float32)
    z = np.stack([wl.gaussian((dv, 3, H, W), 50 + a) for a in range(A)]).astype(np.float32)
    return tps, cams, m, x_t, z


def _dev(tps, cams, m, dtype):
    dt = torch.bfloat16 if dtype == "bf16" else torch.float32
    tp = torch.from_numpy(np.stack(tps)).cuda().to(dt).contiguous()
    intr = torch.from_numpy(np.stack([c.intrinsics for c in cams])).cuda().contiguous()
    c2w = torch.from_numpy(np.stack([c.c2w for c in cams])).cuda().contiguous()
    return tp, intr, c2w, api.DeviceMLP.from_host(m, dtype, "cuda")


@pytest.mark.parametrize("engine,dtype", [("tcgen05", "bf16"), ("simt", "bf16"), ("simt", "f32")])
def test_batched_equals_single_asset_calls(engine, dtype):
    A, H, W = 3, 20, 24
    tps, cams, m, x_t, z = _assets(A, dtype=dtype)
    tp, intr, c2w, mlp = _dev(tps, cams, m, dtype)
    xt, zz = torch.from_numpy(x_t).cuda(), torch.from_numpy(z).cuda()
    kw = dict(samples_per_ray=40, term_eps=1e-4, engine=engine)
    xp, rgb, alpha = api.dmv3d_render_ddim_step_batched(tp, intr, c2w, H, W, mlp, AB, 500, 480, xt,
                                                        z=zz, eta=1.0, keep_mask=[0, 1], **kw)
    for a in range(A):
        xp1, rgb1, al1 = api.dmv3d_render_ddim_step(tp[a], intr[a], c2w[a], H, W, mlp, AB, 500, 480,
                                                    xt[a], z=zz[a], eta=1.0, keep_mask=[0, 1], **kw)
        assert torch.equal(rgb[a], rgb1) and torch.equal(alpha[a], al1) and torch.equal(xp[a], xp1), a


def test_batched_tc_against_oracle_per_asset():
    A, H, W = 3, 20, 24
    tps, cams, m, x_t, _ = _assets(A)
    tp, intr, c2w, mlp = _dev(tps, cams, m, "bf16")
    xt = torch.from_numpy(x_t).cuda()
    xp, rgb, alpha = api.dmv3d_render_ddim_step_batched(tp, intr, c2w, H, W, mlp, AB, 980, 960, xt,
                                                        samples_per_ray=48, term_eps=1e-4,
                                                        engine="tcgen05")
    rgb, alpha, xp = rgb.cpu().numpy(), alpha.cpu().numpy(), xp.cpu().numpy()
    for a in range(A):
        orgb, oalpha = oracle.render_views(tps[a], cams[a], m, 48)
        oxp = oracle.ddim_step(oracle.cosine_alpha_bar(), 980, 960, x_t[a], orgb[:2])
        assert np.abs(rgb[a] - orgb).max() < 2e-2 and np.abs(alpha[a] - oalpha).max() < 1e-2
        assert np.abs(xp[a] - oxp).max() < ddim_tol(AB, 980, 960, 2e-2)


@pytest.mark.parametrize("agg,mode", [("concat", "align_corners"), ("mean", "halfpixel_zeros")])
def test_batched_tc_variants_equal_single(agg, mode):
    """The K0 paths that keep per-asset state: concat (per-plane projections) and the
    half-pixel mode's bias row, one per asset."""
    A, H, W, C = 2, 16, 16, 16
    tps, cams, m, x_t, _ = _assets(A, C=C, H=H, W=W)
    if agg == "concat":
        m = wl.bf16_mlp(wl.random_mlp(3 * C, 64, 3, seed=7))
    tp, intr, c2w, mlp = _dev(tps, cams, m, "bf16")
    kw = dict(samples_per_ray=32, engine="tcgen05", agg=agg, sample_mode=mode)
    rgb, alpha = api.dmv3d_render_views_batched(tp, intr, c2w, H, W, mlp, **kw)
    for a in range(A):
        r1, a1 = api.dmv3d_render_views(tp[a], intr[a], c2w[a], H, W, mlp, **kw)
        assert torch.equal(rgb[a], r1) and torch.equal(alpha[a], a1)


@pytest.mark.parametrize("engine", ["tcgen05", "simt"])
def test_ddim_only_renders_only_ddim_views(engine):
    H, W = 24, 20
    tps, cams, m, x_t, _ = _assets(1, H=H, W=W, dv=2, nv=2)
    tp, intr, c2w, mlp = _dev(tps, cams, m, "bf16")
    xt = torch.from_numpy(x_t[0]).cuda()
    kw = dict(samples_per_ray=32, term_eps=1e-4, engine=engine)
    full, _, _ = api.dmv3d_render_ddim_step(tp[0], intr[0], c2w[0], H, W, mlp, AB, 980, 960, xt, **kw)
    cnt = torch.zeros(8, dtype=torch.int64, device="cuda")
    only, rgb, alpha = api.dmv3d_render_ddim_step(tp[0], intr[0], c2w[0], H, W, mlp, AB, 980, 960, xt,
                                                  want_rgb=False, want_alpha=False, counters=cnt,
                                                  **kw)
    assert rgb is None and alpha is None and torch.equal(full, only)
    assert int(cnt[3]) == 2 * H * W  # the 2 novel views were not marched


@pytest.mark.parametrize("engine", ["tcgen05", "simt"])
def test_skip_kept_views(engine):
    H, W = 20, 20
    tps, cams, m, x_t, _ = _assets(1, H=H, W=W, dv=3, nv=1)
    tp, intr, c2w, mlp = _dev(tps, cams, m, "bf16")
    xt = torch.from_numpy(x_t[0]).cuda()
    kw = dict(samples_per_ray=32, term_eps=1e-4, engine=engine, keep_mask=[1, 0, 0])
    ref_xp, ref_rgb, _ = api.dmv3d_render_ddim_step(tp[0], intr[0], c2w[0], H, W, mlp, AB, 980, 960,
                                                    xt, **kw)
    rgb0 = torch.full((4, 3, H, W), -7.0, device="cuda")
    cnt = torch.zeros(8, dtype=torch.int64, device="cuda")
    xp, rgb, _ = api.dmv3d_render_ddim_step(tp[0], intr[0], c2w[0], H, W, mlp, AB, 980, 960, xt,
                                            rgb=rgb0, skip_kept_views=True, counters=cnt, **kw)
    assert torch.equal(xp, ref_xp)  # kept view: x_t copied either way
    assert torch.equal(xp[0], xt[0])
    assert bool((rgb[0] == -7.0).all())  # not rendered
    assert torch.equal(rgb[1:], ref_rgb[1:])
    assert int(cnt[3]) == 3 * H * W
