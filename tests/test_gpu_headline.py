"""Parity at the headline size (SURVEY.md §4 layer 4: "a seeded subset of 65,536 rays
plus full-image invariants"), in the launch configuration bench.py times: the cfg3 fused
step (8 views 256^2, R=64, C=80, N=128, MLP 80-64-64-64-4, term_eps 1e-4, DDIM on the 4
input views at t = 980 -> 960) on the tensor cores.

* 65,536 seeded rays against the fp64 oracle (all host cores): rgb within 2e-2, alpha
  within 1e-2 (north_star's bf16 tensor-core bar; the termination error <= term_eps is
  far inside it), x_{t-1} of the DDIM views within the DDIM map's Lipschitz bound of it;
* the full image against the fp32 SIMT engine (same bf16 inputs): every pixel within
  the same bar; the same hit / processed-ray counts.
"""
import os

import numpy as np
import pytest
import torch

import oracle
from paper_2605_18052_b200 import api, schedule
from paper_2605_18052_b200 import workloads as wl

from helpers import ddim_tol, dev_workload, flat_ids, pick

pytestmark = pytest.mark.gpu
RGB_TOL, ALPHA_TOL = 2e-2, 1e-2
T, TP = 980, 960


@pytest.fixture(scope="module")
def cfg3():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    w = wl.make_workload("cfg3")
    tp, intr, c2w, mlp = dev_workload(w)
    x_t = torch.from_numpy(wl.gaussian((4, 3, 256, 256), wl.SEED_XT)).cuda()
    return w, tp, intr, c2w, mlp, x_t


def _step(cfg, engine):
    w, tp, intr, c2w, mlp, x_t = cfg
    cnt = torch.zeros(8, dtype=torch.int64, device="cuda")
    xp, rgb, alpha = api.dmv3d_render_ddim_step(tp, intr, c2w, 256, 256, mlp, schedule.cosine_alpha_bar(),
                                                T, TP, x_t, samples_per_ray=128, term_eps=1e-4,
                                                engine=engine, counters=cnt)
    torch.cuda.synchronize()
    return xp.cpu().numpy(), rgb.cpu().numpy(), alpha.cpu().numpy(), cnt.cpu().numpy()


def test_cfg3_step_65536_rays_vs_oracle(cfg3):
    w = cfg3[0]
    xp, rgb, alpha, cnt = _step(cfg3, "tcgen05")
    ids = flat_ids(8, 256, 256, 65536, seed=65536)
    orgb, oalpha = oracle.render_rays(w.triplane, w.cameras, w.mlp, 128, ids,
                                      threads=os.cpu_count() or 1)
    g_rgb, g_alpha = pick(rgb, alpha, ids, 256, 256)
    e_rgb, e_a = np.abs(g_rgb - orgb).max(), np.abs(g_alpha - oalpha).max()
    print(f"{len(ids)} rays: max|rgb-oracle|={e_rgb:.3g} max|alpha-oracle|={e_a:.3g}")
    assert e_rgb < RGB_TOL and e_a < ALPHA_TOL
    # x_{t-1} at the sampled pixels of the DDIM (input) views, oracle DDIM of the oracle rgb
    ab = oracle.cosine_alpha_bar()
    sel = ids < 4 * 256 * 256
    v, pix = ids[sel] // 65536, ids[sel] % 65536
    i, j = pix // 256, pix % 256
    x_t = wl.gaussian((4, 3, 256, 256), wl.SEED_XT)
    img = np.zeros((4, 3, 256, 256))
    img[v, :, i, j] = orgb[sel]
    oxp = oracle.ddim_step(ab, T, TP, x_t, img)
    e_x = np.abs(xp[v, :, i, j] - oxp[v, :, i, j]).max()
    assert e_x < ddim_tol(ab, T, TP, RGB_TOL)
    assert cnt[3] == w.num_rays


def test_cfg3_step_full_image_tc_vs_simt(cfg3):
    xa, ra, aa, ca = _step(cfg3, "tcgen05")
    xb, rb, ab_, cb = _step(cfg3, "simt")
    e_rgb, e_a = np.abs(ra - rb).max(), np.abs(aa - ab_).max()
    print(f"full image: max|rgb tc-simt|={e_rgb:.3g} max|alpha tc-simt|={e_a:.3g} "
          f"mean|rgb|={np.abs(ra - rb).mean():.3g}")
    assert e_rgb < RGB_TOL and e_a < ALPHA_TOL
    ab = schedule.cosine_alpha_bar()
    assert np.abs(xa - xb).max() < ddim_tol(ab, T, TP, RGB_TOL)
    assert ca[0] == cb[0] and ca[3] == cb[3]  # hit rays, processed rays: geometry is exact
