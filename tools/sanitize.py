"""Small invocations of every CUDA entry point for compute-sanitizer:
    compute-sanitizer --tool memcheck|racecheck|synccheck|initcheck python tools/sanitize.py
Tensor-core and SIMT renders (fused DDIM, ray range, tiles), backward on both engines,
density grid on both engines, standalone DDIM, Plucker map, stage-level debug entries."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from paper_2605_18052_b200 import api, schedule  # noqa: E402
from paper_2605_18052_b200 import workloads as wl  # noqa: E402
from helpers import dev_workload  # noqa: E402

H, W, N = 12, 10, 24
tp = wl.round_to_bf16(wl.blob_triplane(12, 32, seed=2, kappa=6.0))
m = wl.bf16_mlp(wl.blob_mlp(32, 64, 4, seed=3))
cams = wl.concat_cameras(wl.input_cameras(H, W, 2), wl.novel_cameras(H, W, 2, seed=4))
ab = schedule.cosine_alpha_bar()
for dtype in ("bf16", "f32"):
    t, intr, c2w, mlp = dev_workload(wl.Workload("san", tp, cams, m, N, dtype))
    engines = ("tcgen05", "simt") if dtype == "bf16" else ("simt",)
    x_t = torch.from_numpy(wl.gaussian((2, 3, H, W), 4)).cuda()
    g = torch.randn((4, 3, H, W), device="cuda")
    for e in engines:
        xp, rgb, alpha = api.dmv3d_render_ddim_step(t, intr, c2w, H, W, mlp, ab, 980, 960, x_t,
                                                    samples_per_ray=N, engine=e, term_eps=1e-4)
        api.dmv3d_render_views(t, intr, c2w, H, W, mlp, samples_per_ray=N, engine=e,
                               ray_range=(37, 3 * H * W - 5))
        api.dmv3d_render_views(t, intr, c2w, H, W, mlp, samples_per_ray=N, engine=e, tiles=(8, 1, 3))
        api.dmv3d_render_backward(t, intr, c2w, H, W, mlp, g, alpha, samples_per_ray=N, engine=e)
        api.dmv3d_render_backward(t, intr, c2w, H, W, mlp, g, None, samples_per_ray=N, engine=e,
                                  term_eps=1e-3, fwd=(rgb, alpha))
        api.dmv3d_density_grid(t, mlp, 13, engine=e)
    api.dmv3d_ddim_step(ab, 500, 480, x_t, rgb[:2].contiguous(), torch.randn_like(x_t), eta=0.5)
    if dtype == "bf16":
        # round 2: SiLU / softplus hidden layers on the tensor cores, range flags, batched step
        for act in (1, 2):
            m2 = wl.bf16_mlp(wl.blob_mlp(32, 64, 4, seed=3))
            m2.hidden_act = act
            api.dmv3d_render_views(t, intr, c2w, H, W, api.DeviceMLP.from_host(m2, "bf16", "cuda"),
                                   samples_per_ray=N, engine="tcgen05")
        api.dmv3d_range_flags()
        tb = torch.stack([t, t]).contiguous()
        xb = torch.stack([x_t, x_t]).contiguous()
        api.dmv3d_render_ddim_step_batched(tb, torch.stack([intr, intr]), torch.stack([c2w, c2w]), H, W,
                                           mlp, ab, 980, 960, xb, samples_per_ray=N, engine="tcgen05",
                                           term_eps=1e-4)
# interleaved-tile merge: pack two ranks' tiles, unpack (ragged 12x10 image, T = 8)
nmax = api.tiles_per_rank(4, H, W, 8, 2)
g3 = torch.zeros((2 * nmax, 3, 8, 8), device="cuda")
g1 = torch.zeros((2 * nmax, 8, 8), device="cuda")
gx = torch.zeros((2 * nmax, 3, 8, 8), device="cuda")
for r in range(2):
    b = slice(r * nmax, (r + 1) * nmax)
    api.dmv3d_tiles_pack(intr, c2w, H, W, 8, r, 2, rgb, alpha, xp, g3[b], g1[b], gx[b], 2)
api.dmv3d_tiles_unpack(intr, c2w, H, W, 8, 2, g3, g1, gx, torch.empty_like(rgb), torch.empty_like(alpha),
                       torch.empty_like(xp), 2)
api.dmv3d_plucker_rays(intr, c2w, H, W)
for rpt in ("1", "2", "4"):  # every store width of the Plucker kernel, with a cut ray range
    os.environ["DMV3D_PLUCKER_RPT"] = rpt
    api.dmv3d_plucker_rays(intr, c2w, H, W, ray_range=(8, 4 * H * W - 4))
os.environ.pop("DMV3D_PLUCKER_RPT")
pts = torch.rand((100, 3), device="cuda") * 2 - 1
api.dmv3d_debug_sample_features(t, pts)
api.dmv3d_debug_decode(t, mlp, pts)
torch.cuda.synchronize()
print("sanitize workload done")
