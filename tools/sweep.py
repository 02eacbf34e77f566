#!/usr/bin/env python
"""Ray-count scaling sweep (BASELINE.json configs[4]): one fused render + DDIM step
of a 3x64x64x80 bf16 asset at image sizes 64^2..512^2 and 4..32 views (4 input views
DDIM-updated, the rest novel), tensor-core engine, N = 128, term_eps = 1e-4.

    python tools/sweep.py [--steps K] [--warmup W] [--out profiles/r01_sweep.jsonl]

Per point: rays/s and evaluated samples/s from CUDA events around each step (L2
flushed between steps), the render kernel's own duration (dmv3d_timer) and its
tensor roofline fraction (27,136 MLP FLOP per evaluated sample / measured bf16 peak).
Single GPU: the sweep is per-GPU work; multi-GPU runs shard assets (bench.py).
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

MLP_FLOPS = 2 * (80 * 64 + 2 * 64 * 64 + 64 * 4)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--sizes", default="64,128,256,512")
    ap.add_argument("--views", default="4,8,16,32")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_sweep.jsonl"))
    args = ap.parse_args()

    import torch
    from paper_2605_18052_b200 import api, schedule
    from paper_2605_18052_b200 import workloads as wl

    dev = torch.device("cuda", 0)
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 1590.0
    tp_h = wl.round_to_bf16(wl.blob_triplane(64, 80))
    m_h = wl.bf16_mlp(wl.blob_mlp(80, 64, 4))
    tp = torch.from_numpy(tp_h).to(dev).to(torch.bfloat16).contiguous()
    mlp = api.DeviceMLP.from_host(m_h, "bf16", dev)
    ab = schedule.cosine_alpha_bar()
    pairs = schedule.ddim_pairs(50, 1000)
    flush = torch.empty((256 << 20) // 4, device=dev)
    stream = torch.cuda.current_stream(dev)
    rows = []
    for S in [int(x) for x in args.sizes.split(",")]:
        for V in [int(x) for x in args.views.split(",")]:
            cams = wl.input_cameras(S, S, 4)
            if V > 4:
                cams = wl.concat_cameras(cams, wl.novel_cameras(S, S, V - 4, seed=wl.SEED_CAMERAS))
            intr = torch.from_numpy(cams.intrinsics).to(dev)
            c2w = torch.from_numpy(cams.c2w).to(dev)
            xa = torch.from_numpy(wl.gaussian((4, 3, S, S), wl.SEED_XT)).to(dev)
            xb = torch.empty_like(xa)
            rgb = torch.empty((V, 3, S, S), device=dev)
            alpha = torch.empty((V, S, S), device=dev)
            cnt = torch.zeros(8, dtype=torch.int64, device=dev)
            timer = api.Timer()

            def step(i, x_in, x_out, counters=None, tm=None):
                t, t_prev = pairs[i % len(pairs)]
                api.dmv3d_render_ddim_step(tp, intr, c2w, S, S, mlp, ab, t, t_prev, x_in, None, 0.0,
                                           x_prev=x_out, rgb=rgb, alpha=alpha, samples_per_ray=128,
                                           term_eps=1e-4, engine="tcgen05", counters=counters,
                                           timer=tm)

            for i in range(args.warmup):
                step(i, xa, xb, cnt if i == 0 else None)
                xa, xb = xb, xa
            torch.cuda.synchronize()
            c = cnt.cpu().numpy().astype(np.float64)
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                  for _ in range(args.steps)]
            for k in range(args.steps):
                flush.zero_()
                ev[k][0].record(stream)
                step(args.warmup + k, xa, xb, tm=timer)
                ev[k][1].record(stream)
                xa, xb = xb, xa
            torch.cuda.synchronize()
            ms = np.array([a.elapsed_time(b) for a, b in ev])
            k_ms, n = timer.read()
            kern = k_ms / max(n, 1)
            rays = V * S * S
            row = {"size": S, "views": V, "rays": rays, "ms_per_step": float(ms.mean()),
                   "rays_per_s": rays / (ms.mean() / 1e3),
                   "samples_per_s_evaluated": c[1] / (ms.mean() / 1e3),
                   "evaluated_fraction": c[1] / (rays * 128.0), "kernel_ms": kern,
                   "tensor_frac": c[1] * MLP_FLOPS / (kern / 1e3) / 1e12 / peak}
            timer.close()
            rows.append(row)
            print(json.dumps(row), flush=True)
    with open(args.out, "w") as f:
        for r in rows:
            f.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
