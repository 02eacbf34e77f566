#!/usr/bin/env python
"""Throughput + roofline of the SURVEY §8(f) rows beyond the headline step
(one JSON line each; CUDA-event timing around the library's own kernel via
dmv3d_timer, warm-up 3, L2 flushed between reps):

  f1  renderer backward   rays/s  (8 views 128^2 training crops, N=128, C=80)
  f2  Plucker ray map     rays/s  (8 views 256^2)            HBM roofline
  f3  density grid        points/s (128^3, C=80 MLP)          FP32-pipe roofline

    python tools/bench_rows.py [--reps 10]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2605_18052_b200 import api  # noqa: E402
from paper_2605_18052_b200 import workloads as wl  # noqa: E402

FP32_PEAK = 148 * 128 * 2 * 1.965e9 / 1e12  # 74.4 TFLOP/s


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    return json.load(open(p)) if os.path.exists(p) else {"hbm_gbs": 6650.0}


def timed(fn, reps, flush, clean=False):
    """Mean kernel ms over `reps` launches, L2 flushed before each: by writing the 256 MiB
    buffer (default), or -- `clean` -- by reading it, which leaves L2 holding clean lines,
    so a write-only kernel is not charged the write-back of the flush's own dirty lines."""
    timer = api.Timer()
    for _ in range(3):
        fn(None)
    torch.cuda.synchronize()
    timer.reset()
    for _ in range(reps):
        if clean:
            flush.sum()
        else:
            flush.zero_()
        fn(timer)
    torch.cuda.synchronize()
    ms, n = timer.read()
    return ms / max(n, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--rows", default="f1,f2,f3", help="comma list of rows to measure")
    args = ap.parse_args()
    dev = torch.device("cuda")
    flush = torch.empty(64 << 20, device=dev)
    pk = peaks()
    out = []

    # f2: Plucker ray map at 8 views 256^2 and 32 views 512^2 (201 MB written)
    import ctypes as ct
    rows = set(args.rows.split(","))
    for V, S in (((8, 256), (32, 512)) if "f2" in rows else ()):
        cams = wl.concat_cameras(wl.input_cameras(S, S, 4), wl.novel_cameras(S, S, V - 4))
        intr = torch.from_numpy(cams.intrinsics).to(dev)
        c2w = torch.from_numpy(cams.c2w).to(dev)
        pl = torch.empty((V, 6, S, S), device=dev)

        def f2(timer):
            c = api.cameras_struct(intr, c2w, S, S)
            o = api.opts_struct(samples_per_ray=1, timer=timer)
            api._abi.check(api._abi.lib().dmv3d_plucker_rays(ct.byref(c), ct.byref(o), pl.data_ptr(),
                                                             api._stream(dev)))
        rays = V * S * S
        for clean in (False, True):
            ms = timed(f2, args.reps, flush, clean)
            gbs = rays * 24 / (ms / 1e3) / 1e9
            out.append({"row": "f2 plucker ray map", "config": f"{V} views {S}^2", "metric": "rays/s",
                        "value": rays / (ms / 1e3), "kernel_ms": ms,
                        "l2_flush": "read 256 MiB (L2 clean)" if clean else
                                    "write 256 MiB (L2 dirty: the flush's write-backs land in the kernel)",
                        "roofline": {"bound": "hbm", "achieved": gbs, "peak": pk["hbm_gbs"], "unit": "GB/s",
                                     "frac": gbs / pk["hbm_gbs"], "algorithmic": "24 B written per ray"}})

    # f3: density grid 128^3, C = 80, L = 4 (bf16 storage, fp32 SIMT decode)
    w = wl.make_workload("cfg3")
    tp = torch.from_numpy(w.triplane).to(dev).to(torch.bfloat16)
    mlp = api.DeviceMLP.from_host(w.mlp, "bf16", dev)
    G = 128

    for engine in (("simt", "tcgen05") if "f3" in rows else ()):
        def f3(timer):
            api.dmv3d_density_grid(tp, mlp, G, timer=timer, engine=engine)
        ms = timed(f3, args.reps, flush)
        pts = G ** 3
        if engine == "simt":
            fl = pts * (27136 + 1920) / (ms / 1e3) / 1e12
            roof = {"bound": "alu", "achieved": fl, "peak": FP32_PEAK, "unit": "TFLOP/s",
                    "frac": fl / FP32_PEAK,
                    "algorithmic": "(27,136 MLP + 1,920 gather) FLOP per point"}
        else:
            fl = pts * 27136 / (ms / 1e3) / 1e12
            roof = {"bound": "tensor", "achieved": fl, "peak": pk.get("bf16_tflops", 1590.0),
                    "unit": "TFLOP/s", "frac": fl / pk.get("bf16_tflops", 1590.0),
                    "algorithmic": "27,136 MLP FLOP per point"}
        out.append({"row": f"f3 density grid ({engine})", "metric": "points/s",
                    "value": pts / (ms / 1e3), "kernel_ms": ms,
                    "config": f"128^3 grid, C=80, MLP 80-64-64-64-4, bf16 storage, {engine}",
                    "roofline": roof})

    if "f1" not in rows and "f1tc" not in rows:
        for line in out:
            print(json.dumps(line))
        return
    # f1: renderer backward, 8 views of 128^2 training crops, N = 128
    cams = wl.concat_cameras(wl.input_cameras(128, 128, 4), wl.novel_cameras(128, 128, 4))
    intr = torch.from_numpy(cams.intrinsics).to(dev)
    c2w = torch.from_numpy(cams.c2w).to(dev)
    g = torch.randn((8, 3, 128, 128), device=dev)
    gA = torch.randn((8, 128, 128), device=dev)

    rays = 8 * 128 * 128
    if "f1" in rows:  # the fp32 SIMT backward (slow: skipped by --rows f1tc)
        def f1(timer):
            api.dmv3d_render_backward(tp, intr, c2w, 128, 128, mlp, g, gA, samples_per_ray=128,
                                      timer=timer)
        ms = timed(f1, max(3, args.reps // 3), flush)
        rays = 8 * 128 * 128
        # algorithmic work per sample: two forward MLP+gather passes, dL/dh (MLP^T), dW (outer
        # products) and the gather transpose
        per = 2 * (27136 + 1920) + 27136 + 27136 + 1920
        hitfrac = 0.95
        fl = rays * hitfrac * 128 * per / (ms / 1e3) / 1e12
        out.append({"row": "f1 renderer backward", "metric": "rays/s", "value": rays / (ms / 1e3),
                    "kernel_ms": ms, "config": "8 views 128^2, N=128, C=80, L=4, fp32 SIMT, atomics",
                    "roofline": {"bound": "alu", "achieved": fl, "peak": FP32_PEAK, "unit": "TFLOP/s",
                                 "frac": fl / FP32_PEAK,
                                 "algorithmic": f"{per} FLOP per sample x ~0.95 hit x 128 samples"}})

    # f1 on the tensor cores (engine tcgen05): same workload; whole call (memset, K0
    # projection, the backward kernel, dF / dW0 maps) and the backward kernel alone
    hit = api.dmv3d_debug_ray_geometry(intr, c2w, 128, 128)[2]
    samples = int(hit.sum().item()) * 128

    def f1tc(timer):
        api.dmv3d_render_backward(tp, intr, c2w, 128, 128, mlp, g, gA, samples_per_ray=128,
                                  timer=timer, engine="tcgen05")
    k_ms = timed(f1tc, args.reps, flush)

    def call_time(fn):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        tot = 0.0
        for _ in range(args.reps):
            flush.zero_()
            e0.record()
            fn(None)
            e1.record()
            torch.cuda.synchronize()
            tot += e0.elapsed_time(e1)
        return tot / args.reps
    call_ms = call_time(f1tc)
    # training-step form: the forward render (term_eps 0) is already there, its rgb /
    # alpha replace the backward's first march (opts.fwd_rgb / fwd_alpha)
    rgb, alpha = api.dmv3d_render_views(tp, intr, c2w, 128, 128, mlp, samples_per_ray=128,
                                        engine="tcgen05")

    def f1tc_fwd(timer):
        api.dmv3d_render_backward(tp, intr, c2w, 128, 128, mlp, g, gA, samples_per_ray=128,
                                  timer=timer, engine="tcgen05", fwd=(rgb, alpha))

    def fwd_only(timer):
        api.dmv3d_render_views(tp, intr, c2w, 128, 128, mlp, rgb=rgb, alpha=alpha,
                               samples_per_ray=128, engine="tcgen05", timer=timer)
    kf_ms = timed(f1tc_fwd, args.reps, flush)
    callf_ms = call_time(f1tc_fwd)
    fwd_ms = call_time(fwd_only)
    # algorithmic work per sample: forward MLP + its transpose (dL/dh) + the weight
    # gradients, 3 x 27,136 FLOP (the implementation's extra forward pass is not counted)
    per_tc = 3 * 27136
    fl = samples * per_tc / (k_ms / 1e3) / 1e12
    bf = pk.get("bf16_tflops", 1654.5)
    out.append({"row": "f1 renderer backward (tcgen05)", "metric": "rays/s",
                "value": rays / (call_ms / 1e3), "call_ms": call_ms, "kernel_ms": k_ms,
                "samples_per_s": samples / (call_ms / 1e3),
                "config": "8 views 128^2, N=128, C=80, L=4, bf16 storage, fp16 MMAs",
                "roofline": {"bound": "tensor", "achieved": fl, "peak": bf, "unit": "TFLOP/s",
                             "frac": fl / bf, "kernel": "render_bwd_tc_kernel",
                             "algorithmic": f"{per_tc} FLOP per sample x {samples} hit samples"}})
    fl2 = samples * per_tc / (kf_ms / 1e3) / 1e12
    out.append({"row": "f1 renderer backward (tcgen05, given the forward's rgb/alpha)",
                "metric": "rays/s", "value": rays / (callf_ms / 1e3), "call_ms": callf_ms,
                "kernel_ms": kf_ms, "forward_render_ms": fwd_ms,
                "forward_plus_backward_rays_per_s": rays / ((fwd_ms + callf_ms) / 1e3),
                "config": "as above; opts.fwd_rgb / fwd_alpha from a term_eps = 0 forward",
                "roofline": {"bound": "tensor", "achieved": fl2, "peak": bf, "unit": "TFLOP/s",
                             "frac": fl2 / bf, "kernel": "render_bwd_tc_kernel",
                             "algorithmic": f"{per_tc} FLOP per sample x {samples} hit samples"}})
    # training with early ray termination (term_eps = 1e-4 in the forward and the backward)
    cnt = torch.zeros(8, dtype=torch.int64, device=dev)
    rgb_t, alpha_t = api.dmv3d_render_views(tp, intr, c2w, 128, 128, mlp, samples_per_ray=128,
                                            engine="tcgen05", term_eps=1e-4, counters=cnt)

    def f1tc_term(timer):
        api.dmv3d_render_backward(tp, intr, c2w, 128, 128, mlp, g, gA, samples_per_ray=128,
                                  timer=timer, engine="tcgen05", term_eps=1e-4, fwd=(rgb_t, alpha_t))
    kt_ms = timed(f1tc_term, args.reps, flush)
    callt_ms = call_time(f1tc_term)
    ev = int(cnt[1].item())  # samples the terminated forward evaluated (= the backward's)
    fl3 = ev * per_tc / (kt_ms / 1e3) / 1e12
    out.append({"row": "f1 renderer backward (tcgen05, term_eps 1e-4, given the forward)",
                "metric": "rays/s", "value": rays / (callt_ms / 1e3), "call_ms": callt_ms,
                "kernel_ms": kt_ms, "evaluated_samples": ev,
                "config": "as above; forward and backward stop a ray once T < 1e-4",
                "roofline": {"bound": "tensor", "achieved": fl3, "peak": bf, "unit": "TFLOP/s",
                             "frac": fl3 / bf, "kernel": "render_bwd_tc_kernel",
                             "algorithmic": f"{per_tc} FLOP per evaluated sample x {ev}"}})
    for line in out:
        print(json.dumps(line))


if __name__ == "__main__":
    main()
