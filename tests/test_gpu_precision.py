"""The tensor-core engine's precision contract (include/dmv3d.h, DMV3D_ENGINE_TCGEN05):

* SiLU and softplus hidden layers (reading A5; PAPER.md:71 leaves the MLP form open) run
  on the tensor cores and match the oracle within the bf16 tensor-core bar;
* fp16 range guard: a projected triplane or an activation beyond +-65504 is not clamped
  silently -- the call's range flags report it (bit 0: G, bit 1: activation) and the
  counters[6] slot counts the non-finite samples; an in-range call reports 0;
* dmv3d_select_engine tells which engine AUTO runs (no silent ~20x slower fallback).
"""
import numpy as np
import pytest
import torch

import oracle
from paper_2605_18052_b200 import api, schedule
from paper_2605_18052_b200 import workloads as wl

from helpers import dev_workload

pytestmark = pytest.mark.gpu
RGB_TOL, ALPHA_TOL = 2e-2, 1e-2


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _wl(act=0, C=32, L=4, H=24, W=20, N=64, seed=11, scale_tp=1.0, w1_scale=1.0):
    tp = wl.blob_triplane(32, C, seed) * scale_tp
    m = wl.blob_mlp(C, 64, L, seed + 1)
    m.hidden_act = act
    if w1_scale != 1.0:
        m.weights[1] = m.weights[1] * np.float32(w1_scale)
    tp, m = wl.round_to_bf16(tp.astype(np.float32)), wl.bf16_mlp(m)
    cams = wl.concat_cameras(wl.input_cameras(H, W, 2), wl.novel_cameras(H, W, 1, seed=seed + 2))
    return wl.Workload("prec", tp, cams, m, N, "bf16")


def _render(w, **kw):
    tp, intr, c2w, mlp = dev_workload(w)
    H, W = w.cameras.height, w.cameras.width
    cnt = torch.zeros(8, dtype=torch.int64, device="cuda")
    rgb, alpha = api.dmv3d_render_views(tp, intr, c2w, H, W, mlp, samples_per_ray=w.samples_per_ray,
                                        term_eps=1e-4, engine="tcgen05", counters=cnt, **kw)
    flags = api.dmv3d_range_flags()
    return rgb.cpu().numpy(), alpha.cpu().numpy(), flags, cnt.cpu().numpy()


@pytest.mark.parametrize("act", [1, 2], ids=["silu", "softplus"])
def test_tc_hidden_activations_match_oracle(act):
    w = _wl(act=act)
    rgb, alpha, flags, cnt = _render(w)
    orgb, oalpha = oracle.render_views(w.triplane, w.cameras, w.mlp, w.samples_per_ray)
    e_rgb, e_a = np.abs(rgb - orgb).max(), np.abs(alpha - oalpha).max()
    print(f"act {act}: max|rgb|={e_rgb:.3g} max|alpha|={e_a:.3g}")
    assert e_rgb < RGB_TOL and e_a < ALPHA_TOL
    assert flags == 0 and cnt[6] == 0


def test_tc_activation_changes_the_result():
    """The template dispatch really switches the activation (SiLU != ReLU here)."""
    r0, _, _, _ = _render(_wl(act=0))
    r1, _, _, _ = _render(_wl(act=1))
    assert np.abs(r0 - r1).max() > 1e-3


def test_range_flags_in_range_is_zero():
    _, _, flags, cnt = _render(_wl())
    assert flags == 0 and cnt[6] == 0


def test_range_flag_projected_triplane_overflow():
    """G = F W0^T + b0 beyond fp16: a triplane scaled by 1e5 (|F| ~ 1e5, W0 ~ 1/sqrt(C))."""
    rgb, _, flags, cnt = _render(_wl(scale_tp=1e5))
    assert flags & api.RANGE_G_OVERFLOW
    assert not np.isfinite(rgb).all() or cnt[6] > 0  # no silent finite clamp downstream


def test_range_flag_activation_overflow():
    """In-range G but layer-1 weights x 1e6: the hidden activations leave fp16 for every
    sample (x 1e4 overflows only near the blob's centre, which early termination never
    reaches)."""
    rgb, _, flags, cnt = _render(_wl(w1_scale=1e6))
    assert flags & api.RANGE_ACT_OVERFLOW
    assert not flags & api.RANGE_G_OVERFLOW
    assert cnt[6] > 0


def test_range_flags_reset_per_call():
    _render(_wl(w1_scale=1e6))
    _, _, flags, _ = _render(_wl())
    assert flags == 0


def test_host_step_range_flags():
    w = _wl(w1_scale=1e6)
    H, W = w.cameras.height, w.cameras.width
    ws = api.Workspace()
    tp = torch.from_numpy(w.triplane).to(torch.bfloat16).pin_memory()
    m = api.DeviceMLP.from_host(w.mlp, "bf16", "cpu")
    x = torch.from_numpy(wl.gaussian((2, 3, H, W), 4)).pin_memory()
    xp = torch.empty_like(x).pin_memory()
    api.dmv3d_render_ddim_step_host(ws, tp, torch.from_numpy(w.cameras.intrinsics),
                                    torch.from_numpy(w.cameras.c2w), H, W, m,
                                    schedule.cosine_alpha_bar(), 500, 480, x, xp,
                                    samples_per_ray=w.samples_per_ray, engine="tcgen05")
    torch.cuda.synchronize()
    assert ws.range_flags() & api.RANGE_ACT_OVERFLOW
    ws.close()


def test_select_engine_reports_auto_choice():
    w = _wl()
    tp, intr, c2w, mlp = dev_workload(w)
    assert api.dmv3d_select_engine(tp, mlp) == "tcgen05"
    assert api.dmv3d_select_engine(tp, mlp, engine="simt") == "simt"
    # hidden 32: the tensor-core engine is hidden-64 only, AUTO takes SIMT -- visibly
    w16 = _wl(C=16)
    tp16, _, _, _ = dev_workload(w16)
    m32 = wl.bf16_mlp(wl.blob_mlp(16, 32, 4, 3))
    assert api.dmv3d_select_engine(tp16, api.DeviceMLP.from_host(m32, "bf16", "cuda")) == "simt"
    # fp32 storage: SIMT
    w32 = wl.Workload("f", w.triplane, w.cameras, w.mlp, 64, "f32")
    tpf, _, _, mf = dev_workload(w32)
    assert api.dmv3d_select_engine(tpf, mf) == "simt"
    with pytest.raises(api._abi.DMV3DError):
        api.dmv3d_select_engine(tpf, mf, engine="tcgen05")
