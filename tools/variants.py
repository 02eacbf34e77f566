#!/usr/bin/env python
"""Throughput + tensor roofline of the SURVEY §8(d) workloads beyond the headline step,
one JSON line each (CUDA-event timing of the render kernel via dmv3d_timer, whole-step
CUDA events around the call, warm-up 3, L2 flushed between steps):

  cfg3_eta1_keep   cfg3 step with eta = 1 (z given) and keep_mask {1,0,0,0} (PAPER.md:91,
                   :1102), rendering every view, and with the kept view's rays skipped
  cfg3_c32         the paper's C = 32 triplane (reading A1)
  cfg3_l2          the L = 2 MLP (reading A5)
  cfg2x8           8 cfg2-sized assets (4 views 128^2 each) in ONE batched launch
  cfg4             BASELINE configs[3] on one GPU: 8 assets x 4 input views 256^2, the
                   50-step DDIM loop (PAPER.md:471; batch 8 per GPU, :2538), one batched
                   launch per step, DDIM views only (no rgb/alpha)
  cachebust        8 assets x 3x256x256x80 bf16 triplanes (240 MiB > L2), 4 input views
                   256^2, one batched step: the regime where HBM can bind

    python tools/variants.py [--only NAME[,NAME]] [--steps 20]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2605_18052_b200 import api, schedule  # noqa: E402
from paper_2605_18052_b200 import workloads as wl  # noqa: E402

TERM_EPS = 1e-4


def flops_per_sample(C, H, L):
    """2 (K H + (L-2) H^2 + 4 H), K = C for the mean aggregation."""
    return 2 * (C * H + (L - 2) * H * H + 4 * H)


def peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    return json.load(open(p)).get("bf16_tflops", 1590.0) if os.path.exists(p) else 1590.0


class Runner:
    def __init__(self, steps):
        self.dev = torch.device("cuda")
        self.flush = torch.empty(64 << 20, device=self.dev)  # 256 MiB
        self.steps = steps
        self.ab = schedule.cosine_alpha_bar()
        self.pairs = schedule.ddim_pairs(50, 1000)

    def measure(self, call, nsteps=None):
        """call(i, timer, counters) -> None.  Returns (step ms, kernel ms, counters)."""
        nsteps = nsteps or self.steps
        cnt = torch.zeros(8, dtype=torch.int64, device=self.dev)
        for i in range(3):
            call(i, None, cnt if i == 0 else None)
        torch.cuda.synchronize()
        timer = api.Timer()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(nsteps)]
        for i in range(nsteps):
            self.flush.zero_()
            ev[i][0].record()
            call(3 + i, timer, None)
            ev[i][1].record()
        torch.cuda.synchronize()
        k_ms, n = timer.read()
        step_ms = float(np.sum([a.elapsed_time(b) for a, b in ev])) / nsteps
        return step_ms, k_ms / max(n, 1), cnt.cpu().numpy().astype(np.float64)


def line(name, rays, step_ms, kernel_ms, c, fps, config, **extra):
    pk = peak()
    achieved = c[1] * fps / (kernel_ms / 1e3) / 1e12
    d = {"variant": name, "config": config, "rays_per_step": rays,
         "rays_per_s": rays / (step_ms / 1e3), "ms_per_step": step_ms, "kernel_ms": kernel_ms,
         "samples_per_s_evaluated": c[1] / (step_ms / 1e3),
         "evaluated_fraction_of_nominal": c[1] / (rays * 128), "hit_fraction": c[0] / max(c[3], 1),
         "mma_row_occupancy": c[1] / c[4] if c[4] else None,
         "mean_blend_k": c[5] / (c[4] / 128) if c[4] else None,
         "roofline": {"bound": "tensor", "achieved": achieved, "peak": pk, "unit": "TFLOP/s",
                      "frac": achieved / pk,
                      "algorithmic": f"{fps} MLP FLOP per evaluated sample x evaluated samples"}}
    d.update(extra)
    print(json.dumps(d), flush=True)
    return d


def cfg3_like(r, name, eta=0.0, keep=None, skip=False):
    w = wl.make_workload(name)
    dev = r.dev
    V, H, W = w.cameras.num_views, w.cameras.height, w.cameras.width
    tp = torch.from_numpy(w.triplane).to(dev).to(torch.bfloat16).contiguous()
    intr = torch.from_numpy(w.cameras.intrinsics).to(dev)
    c2w = torch.from_numpy(w.cameras.c2w).to(dev)
    mlp = api.DeviceMLP.from_host(w.mlp, "bf16", dev)
    x = [torch.from_numpy(wl.gaussian((4, 3, H, W), wl.SEED_XT)).to(dev), torch.empty((4, 3, H, W), device=dev)]
    z = torch.from_numpy(wl.gaussian((4, 3, H, W), wl.SEED_Z)).to(dev) if eta > 0 else None
    rgb = torch.empty((V, 3, H, W), device=dev)
    alpha = torch.empty((V, H, W), device=dev)

    def call(i, timer, cnt):
        t, tp_ = r.pairs[i % len(r.pairs)]
        api.dmv3d_render_ddim_step(tp, intr, c2w, H, W, mlp, r.ab, t, tp_, x[i % 2], z, eta, keep,
                                   x_prev=x[(i + 1) % 2], rgb=rgb, alpha=alpha, samples_per_ray=128,
                                   term_eps=TERM_EPS, engine="tcgen05", counters=cnt, timer=timer,
                                   skip_kept_views=skip)
    return w, V * H * W, call


def batched(r, wname, A, views, res, R=None):
    """A assets of workload `wname` (seeds 100 + a) sharing the MLP; `views` input views."""
    dev = r.dev
    ws = [wl.make_workload(wname, asset=a) for a in range(A)]
    if R is not None:  # re-draw the triplanes at resolution R (cache-busting point)
        tps = [wl.round_to_bf16(wl.blob_triplane(R, ws[0].channels, 100 + a)) for a in range(A)]
    else:
        tps = [w.triplane for w in ws]
    cams = wl.input_cameras(res, res, views)
    tp = torch.from_numpy(np.stack(tps)).to(dev).to(torch.bfloat16).contiguous()
    intr = torch.from_numpy(np.stack([cams.intrinsics] * A)).to(dev)
    c2w = torch.from_numpy(np.stack([cams.c2w] * A)).to(dev)
    mlp = api.DeviceMLP.from_host(ws[0].mlp, "bf16", dev)
    x = [torch.from_numpy(wl.gaussian((A, views, 3, res, res), wl.SEED_XT)).to(dev),
         torch.empty((A, views, 3, res, res), device=dev)]

    def call(i, timer, cnt):
        t, tp_ = r.pairs[i % len(r.pairs)]
        api.dmv3d_render_ddim_step_batched(tp, intr, c2w, res, res, mlp, r.ab, t, tp_, x[i % 2],
                                           x_prev=x[(i + 1) % 2], want_rgb=False, want_alpha=False,
                                           samples_per_ray=128, term_eps=TERM_EPS, engine="tcgen05",
                                           counters=cnt, timer=timer)
    return ws[0], A * views * res * res, call, tp


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="")
    ap.add_argument("--steps", type=int, default=20)
    args = ap.parse_args()
    only = set(filter(None, args.only.split(",")))
    r = Runner(args.steps)
    want = lambda n: not only or n in only  # noqa: E731
    wk = "cfg3: 8 views 256^2, R=64, N=128, H=64, fused DDIM on the 4 input views, term_eps 1e-4"

    if want("cfg3_eta1_keep"):
        for skip in (False, True):
            w, rays, call = cfg3_like(r, "cfg3", eta=1.0, keep=[1, 0, 0, 0], skip=skip)
            s, k, c = r.measure(call)
            line("cfg3_eta1_keep" + ("_skip" if skip else ""), rays, s, k, c, flops_per_sample(80, 64, 4),
                 wk + ", C=80, L=4, eta=1 with z, keep_mask {1,0,0,0}"
                 + (", kept view not rendered (x_{t-1} = x_t, its rgb/alpha untouched)" if skip else ""))
    if want("cfg3_c32"):
        w, rays, call = cfg3_like(r, "cfg3_c32")
        s, k, c = r.measure(call)
        line("cfg3_c32", rays, s, k, c, flops_per_sample(32, 64, 4), wk + ", C=32 (PAPER.md:2537), L=4")
    if want("cfg3_l2"):
        w, rays, call = cfg3_like(r, "cfg3_l2")
        s, k, c = r.measure(call)
        line("cfg3_l2", rays, s, k, c, flops_per_sample(80, 64, 2), wk + ", C=80, L=2 (80-64-4)")
    if want("cfg2x8"):
        w, rays, call, _ = batched(r, "cfg2_bf16", 8, 4, 128)
        s, k, c = r.measure(call)
        line("cfg2x8", rays, s, k, c, flops_per_sample(80, 64, 4),
             "8 cfg2 assets (4 input views 128^2 each, R=64, C=80, L=4) in one batched launch, DDIM "
             "views only")
    if want("cfg4"):
        w, rays, call, _ = batched(r, "cfg3", 8, 4, 256)
        # the whole 50-step loop, one batched launch per step (L2 flushed between steps)
        s, k, c = r.measure(call, nsteps=50)
        line("cfg4", rays, s, k, c, flops_per_sample(80, 64, 4),
             "cfg4: 8 assets (seeds 100-107) x 4 input views 256^2, R=64, C=80, L=4, shared MLP, "
             "the 50-step DDIM grid 980..0 (one batched launch per step, DDIM views only)",
             loop_ms=50 * s, loop_rays_per_s=50 * rays / (50 * s / 1e3))
    if want("cachebust"):
        w, rays, call, tp = batched(r, "cfg3", 8, 4, 256, R=256)
        s, k, c = r.measure(call, nsteps=max(5, args.steps // 4))
        tb = tp.numel() * tp.element_size()
        gb = 8 * (3 * 256 * 256 + 1) * 64 * 2
        line("cachebust", rays, s, k, c, flops_per_sample(80, 64, 4),
             "8 assets x 3x256x256x80 bf16 triplanes (240 MiB), 4 input views 256^2 each, N=128, "
             "L=4, one batched step", triplane_bytes=tb, g_bytes=gb,
             compulsory_hbm_note="K0 reads the triplanes (240 MiB) and writes G (192 MiB); the "
                                 "render kernel reads G once per asset (192 MiB)")


if __name__ == "__main__":
    main()
