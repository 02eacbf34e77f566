#!/usr/bin/env python
"""Per-phase cycle breakdown of render_tc_kernel (one cfg3 step).

    python tools/phases.py            # builds libdmv3d_phases.so (-DDMV3D_PHASES), runs

Every thread of the kernel accumulates clock64 deltas per phase; row 0 of each group
adds them to counters[8..15].  Printed: share of a group's time per phase and cycles
per group per chunk (chunks = group-tiles, from the sample counter / rows).
"""
from __future__ import annotations

import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
PHASES = ["patch setup + first prefetch", "A scatter (sparse blend rows)",
          "blend: cp.async wait + MMA round trip", "prefetch next chunk (geometry, window, staging)",
          "layer epilogues (TMEM ld, ReLU, fp16, TMEM st)", "layer MMA round trips (bar + issue + wait)",
          "head + compositing + loop control", "ray epilogue + next patch fetch"]


def run():
    import numpy as np
    import torch
    from paper_2605_18052_b200 import api, schedule
    from paper_2605_18052_b200 import workloads as wl
    w = wl.make_workload("cfg3")
    dev = torch.device("cuda", 0)
    V, H, W = w.cameras.num_views, w.cameras.height, w.cameras.width
    tp = torch.from_numpy(w.triplane).to(dev).to(torch.bfloat16).contiguous()
    intr = torch.from_numpy(w.cameras.intrinsics).to(dev)
    c2w = torch.from_numpy(w.cameras.c2w).to(dev)
    mlp = api.DeviceMLP.from_host(w.mlp, "bf16", dev)
    ab = schedule.cosine_alpha_bar()
    x = torch.from_numpy(wl.gaussian((4, 3, H, W), wl.SEED_XT)).to(dev)
    for it in range(3):
        cnt = torch.zeros(16, dtype=torch.int64, device=dev)
        api.dmv3d_render_ddim_step(tp, intr, c2w, H, W, mlp, ab, 980, 960, x, None, 0.0,
                                   samples_per_ray=128, term_eps=1e-4, engine="tcgen05",
                                   counters=cnt)
        torch.cuda.synchronize()
    c = cnt.cpu().numpy().astype(np.float64)
    ph = c[8:16]
    groups = 148 * 4
    tot = ph.sum()
    print(f"evaluated samples {c[1]:.0f}; per-group cycles {tot / groups:.0f} "
          f"(= {tot / groups / 1.965e6:.3f} ms at 1965 MHz)")
    for name, v in zip(PHASES, ph):
        print(f"  {100 * v / tot:5.1f}%  {name}")


if __name__ == "__main__":
    if os.environ.get("DMV3D_LIB"):
        run()
    else:
        from paper_2605_18052_b200 import build
        lib = build.build(defines=["DMV3D_PHASES"],
                          lib=os.path.join(ROOT, "paper_2605_18052_b200", "libdmv3d_phases.so"),
                          objdir=os.path.join(ROOT, "paper_2605_18052_b200", "build_phases"))
        env = dict(os.environ, DMV3D_LIB=lib)
        sys.exit(subprocess.call([sys.executable, __file__], env=env))
