#!/usr/bin/env python
"""Per-role phase breakdown of render_ws_kernel (one cfg3 step); run with
DMV3D_LIB=libdmv3d_phases.so (built by tools/phases.py)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GROUP = ["wait full (tile staged)", "blend issue + MMA wait", "MLP layers", "head + composite + publish"]
SAMPLER = ["wait empty (stage free)", "fetch patch (rays) / composited spin", "geometry + bbox + barrier",
           "table + cp.async issue", "A zero + scatter", "cp.async wait + fence + arrive",
           "loop between feeds", "-"]


def run():
    import numpy as np
    import torch
    from paper_2605_18052_b200 import api, schedule
    from paper_2605_18052_b200 import workloads as wl
    w = wl.make_workload("cfg3")
    dev = torch.device("cuda", 0)
    H, W = w.cameras.height, w.cameras.width
    tp = torch.from_numpy(w.triplane).to(dev).to(torch.bfloat16).contiguous()
    intr = torch.from_numpy(w.cameras.intrinsics).to(dev)
    c2w = torch.from_numpy(w.cameras.c2w).to(dev)
    mlp = api.DeviceMLP.from_host(w.mlp, "bf16", dev)
    ab = schedule.cosine_alpha_bar()
    x = torch.from_numpy(wl.gaussian((4, 3, H, W), wl.SEED_XT)).to(dev)
    for it in range(3):
        cnt = torch.zeros(24, dtype=torch.int64, device=dev)
        api.dmv3d_render_ddim_step(tp, intr, c2w, H, W, mlp, ab, 980, 960, x, None, 0.0,
                                   samples_per_ray=128, term_eps=1e-4, engine="tcgen05",
                                   counters=cnt)
        torch.cuda.synchronize()
    c = cnt.cpu().numpy().astype(np.float64)
    tiles = c[4] / 128
    for name, ph, nrole in (("group", c[8:12], 4), ("sampler", c[16:24], 2)):
        tot = ph.sum()
        print(f"{name}: cycles per role instance {tot / (148 * nrole):.0f}; per tile "
              f"{tot / tiles * (1 if name == 'group' else 1):.0f} (summed over instances)")
        for nm, v in zip(GROUP if name == "group" else SAMPLER, ph):
            print(f"  {100 * v / max(tot, 1):5.1f}%  {nm}")


if __name__ == "__main__":
    run()
