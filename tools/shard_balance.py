#!/usr/bin/env python
"""Load balance of the N > 1 splits on one GPU: the cfg3 step's render-kernel time of each
rank's share for P = 2, 4, 8 under the view split (contiguous view blocks, ray ranges)
and the interleaved 16x16 tile split (opts.tile_*), measured one share at a time (CUDA
events of the library's timer, L2 flushed before each).  The step time of a split is the
max over its ranks; mean / max is the split's balance."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_18052_b200 import api, schedule  # noqa: E402
from paper_2605_18052_b200 import workloads as wl  # noqa: E402


def main():
    w = wl.make_workload("cfg3")
    dev = torch.device("cuda")
    V, H, W = 8, 256, 256
    tp = torch.from_numpy(w.triplane).to(dev).to(torch.bfloat16).contiguous()
    intr = torch.from_numpy(w.cameras.intrinsics).to(dev)
    c2w = torch.from_numpy(w.cameras.c2w).to(dev)
    mlp = api.DeviceMLP.from_host(w.mlp, "bf16", dev)
    ab = schedule.cosine_alpha_bar()
    x = torch.from_numpy(wl.gaussian((4, 3, H, W), wl.SEED_XT)).to(dev)
    flush = torch.empty(64 << 20, device=dev)

    def share_ms(**kw):
        timer = api.Timer()
        for it in range(8):
            flush.zero_()
            if it == 3:
                timer.reset()
            api.dmv3d_render_ddim_step(tp, intr, c2w, H, W, mlp, ab, 980, 960, x, samples_per_ray=128,
                                       term_eps=1e-4, engine="tcgen05", timer=timer if it >= 3 else None, **kw)
        torch.cuda.synchronize()
        ms, n = timer.read()
        return ms / n

    full = share_ms()
    print(json.dumps({"split": "none", "P": 1, "ms": [full]}))
    for P in (2, 4, 8):
        per = -(-V // P)
        views = [share_ms(ray_range=(r * per * H * W, min(V, (r + 1) * per) * H * W)) for r in range(P)]
        tiles = [share_ms(tiles=(16, r, P)) for r in range(P)]
        for name, ms in (("views", views), ("tiles", tiles)):
            print(json.dumps({"split": name, "P": P, "ms": ms, "max": max(ms), "mean": float(np.mean(ms)),
                              "balance": float(np.mean(ms) / max(ms)), "speedup_vs_1": full / max(ms)}))


if __name__ == "__main__":
    main()
