#!/usr/bin/env python
"""Benchmark: rays/s of one DMV3D denoise step (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

A step is one fused pass of the whole hot path
over one asset: render 4 input + 4 novel views at 256x256 from a
3x64x64x80 bf16 triplane with N = 128 samples/ray through the shared
80-64-64-64-4 MLP, composite, and apply the DDIM x_{t-1} update to the 4
input views (cfg3).  Steps walk the paper's 50-step DDIM grid 980 -> 0
(PAPER.md:471), feeding x_{t-1} back as the next x_t.  Multi-GPU (torchrun): by default the
ONE asset's views are split across the ranks (strong scaling; PAPER.md:45-46:
every step renders from the current triplane): each step broadcasts the packed triplane +
MLP from rank 0 over NCCL, renders this rank's views and all-gathers rgb / alpha /
x_{t-1} -- all inside the timed region; timing is the max over ranks.  The line also
carries `weak_assets`: one independent asset per rank, no data-path collective.

Prints ONE JSON line on rank 0.  `value` = rays/s over all ranks with inputs
resident in HBM; `e2e` = the same through the host-buffer C-ABI entry
(pinned host in/out copies inside the timed region); `roofline` = the render
kernel's algorithmic MLP FLOPs / its CUDA-event time vs the measured dense
bf16 peak; `cpu_baseline` = the CPU oracle on a bounded sample of the
same workload on this host's cores.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# --config: cfg3 = BASELINE configs[2], the step north_star's target names ("a 4-view +
# novel-view DDIM step at the paper's triplane and image sizes"): the default and the
# headline.  cfg2 = configs[1] (4 input views at 128^2, paper-shaped triplane and MLP).
CONFIGS = {
    "cfg3": ("cfg3",
             "rays/s per denoise-step render (4 input + 4 novel views 256x256, fused DDIM)",
             "cfg3: 4 input + 4 novel views 256x256, triplane 3x64x64x80 bf16, N=128 "
             "midpoint samples/ray, shared MLP 80-64-64-64-4 (ReLU), fused DDIM on the 4 "
             "input views along the 50-step grid 980..0, eta=0, term_eps=1e-4, white bg"),
    "cfg2": ("cfg2_bf16",
             "rays/s per denoise-step render (4 input views 128x128, fused DDIM)",
             "cfg2: 4 input views 128x128, triplane 3x64x64x80 bf16, N=128 midpoint "
             "samples/ray, shared MLP 80-64-64-64-4 (ReLU), fused DDIM on the 4 views along "
             "the 50-step grid 980..0, eta=0, term_eps=1e-4, white bg"),
}
METRIC, WORKLOAD = CONFIGS["cfg3"][1], CONFIGS["cfg3"][2]
MLP_FLOPS_PER_SAMPLE = 2 * (80 * 64 + 2 * 64 * 64 + 64 * 4)  # 27,136
TERM_EPS = 1e-4
L2_FLUSH_BYTES = 256 << 20


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
            "sm_max_mhz": 1965.0}, "fallback"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int, period_ms: int = 50):
        self.gpu = gpu_index
        self.period = period_ms
        self.rows = []
        self._proc = None
        self._t = threading.Thread(target=self._read, daemon=True)

    def _read(self):
        for line in self._proc.stdout:
            parts = [x.strip() for x in line.strip().split(",")]
            if len(parts) >= 6:
                self.rows.append(parts)

    def __enter__(self):
        try:
            self._proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", f"-lms={self.period}"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t.start()
            t0 = time.time()
            while not self.rows and time.time() - t0 < 3.0:  # sampler is live before timing
                time.sleep(0.02)
        except Exception:
            self._proc = None
        return self

    def __exit__(self, *a):
        if self._proc is not None:
            time.sleep(2 * self.period / 1e3)
            self._proc.terminate()
            try:
                self._proc.wait(timeout=5)
            except Exception:
                self._proc.kill()
            self._t.join(timeout=5)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4)
                          if len(r) > 2 + k and r[2 + k].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ------------------------------------------------------------------ CPU oracle leg
def oracle_rate(w, budget_s: float, threads: int, max_rays: int = 524288, seed: int = 7):
    """Oracle rays/s on a bounded random sample of the workload's rays."""
    import oracle
    rng = np.random.default_rng(seed)
    ids = rng.permutation(w.num_rays)[:max_rays]
    done, t0, chunk = 0, time.perf_counter(), 256
    while done < len(ids) and time.perf_counter() - t0 < budget_s:
        oracle.render_rays(w.triplane, w.cameras, w.mlp, w.samples_per_ray, ids[done:done + chunk],
                           threads=threads)
        done += chunk
        chunk = min(chunk * 2, 4096)
    dt = time.perf_counter() - t0
    return done / dt, done, dt


def run_reference(args, rank, world):
    """--impl reference: the CPU oracle as it stands, on this host's cores."""
    if rank != 0:
        return
    from paper_2605_18052_b200 import workloads as wl
    wname, metric, workload = CONFIGS[args.config]
    w = wl.make_workload(wname)
    threads = os.cpu_count() or 1
    rays_per_step = 2048
    import oracle
    rng = np.random.default_rng(11)
    times = []
    for s in range(args.warmup + args.steps):
        ids = rng.choice(w.num_rays, rays_per_step, replace=False)
        t0 = time.perf_counter()
        oracle.render_rays(w.triplane, w.cameras, w.mlp, w.samples_per_ray, ids, threads=threads)
        if s >= args.warmup:
            times.append(time.perf_counter() - t0)
    total = float(np.sum(times))
    value = rays_per_step * len(times) / total
    line = {"impl": "reference", "metric": metric, "value": value, "unit": "rays/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * total / len(times), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload, "rays_per_step_sampled": rays_per_step},
            "cpu_baseline": {"value": value, "unit": "rays/s", "cores": threads, "kind": "oracle",
                             "cpu_model": _cpu_model(),
                             "sample": f"{rays_per_step} random rays of {args.config} per step (of "
                                       f"{w.num_rays}), full 128-sample march, fp64, no early "
                                       "termination"},
            "e2e": {"value": value, "unit": "rays/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU leg
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg3", choices=sorted(CONFIGS),
                    help="cfg3 (default, BASELINE configs[2]) or cfg2 (configs[1])")
    ap.add_argument("--engine", default="auto", choices=["auto", "simt", "tcgen05"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--sustained-s", type=float, default=2.0,
                    help="also time >= this many seconds of steps (sustained clocks); 0: skip")
    ap.add_argument("--share-gpu", action="store_true",
                    help="dry run of the N > 1 path on one GPU: every rank on cuda:0, gloo")
    ap.add_argument("--mode", default="auto",
                    choices=["auto", "assets", "views", "views-p2p", "tiles", "tiles-p2p"],
                    help="auto: views for N > 1; assets: one asset per rank, no data-path "
                         "collective (weak scaling); views: one asset's views split across ranks with an NCCL "
                         "triplane broadcast + all-gather per step (strong scaling); views-p2p: "
                         "the same split, outputs assembled by the render kernel's NVLink peer "
                         "stores into symmetric memory; tiles: one asset's 16x16 ray tiles dealt "
                         "round robin to the ranks, outputs assembled by one all-gather of packed tiles; tiles-p2p: "
                         "the same, assembled by the render kernel's NVLink peer stores")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist

    from paper_2605_18052_b200 import api, schedule
    from paper_2605_18052_b200 import workloads as wl

    if args.mode == "auto":
        args.mode = "views" if world > 1 else "assets"
    gpu = 0 if args.share_gpu else local_rank
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    if world > 1:
        if args.share_gpu:  # NCCL refuses two ranks on one device
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    from paper_2605_18052_b200 import dist as pdist

    # ---- inputs (one asset per rank, seeds 100 + rank), resident in HBM
    views_mode = args.mode in ("views", "views-p2p", "tiles", "tiles-p2p")
    wname, metric, workload = CONFIGS[args.config]
    w = wl.make_workload(wname, asset=rank if (world > 1 and not views_mode) else None)
    V, H, W = w.cameras.num_views, w.cameras.height, w.cameras.width
    DV = w.ddim_views or V  # the DDIM-updated (input) views
    tdt = torch.bfloat16 if w.dtype == "bf16" else torch.float32
    tp = torch.from_numpy(w.triplane).to(dev).to(tdt).contiguous()
    intr = torch.from_numpy(w.cameras.intrinsics).to(dev)
    c2w = torch.from_numpy(w.cameras.c2w).to(dev)
    mlp = api.DeviceMLP.from_host(w.mlp, w.dtype, dev)
    # strong-scaling modes: the triplane and MLP in one buffer, broadcast by rank 0 every step
    asset = pdist.PackedAsset(tp, mlp) if views_mode else None
    ab = schedule.cosine_alpha_bar()
    pairs = schedule.ddim_pairs(50, 1000)
    x0 = torch.from_numpy(wl.gaussian((DV, 3, H, W), wl.SEED_XT)).to(dev)
    xa, xb = x0.clone(), torch.empty_like(x0)
    rgb = torch.empty((V, 3, H, W), device=dev)
    alpha = torch.empty((V, H, W), device=dev)
    flush = torch.empty(L2_FLUSH_BYTES // 4, device=dev)
    counters = torch.zeros(8, dtype=torch.int64, device=dev)
    rays = V * H * W
    stream = torch.cuda.current_stream(dev)

    kernel_timer = api.Timer()

    def sharded(i, x_in, cnt=None, timer=None):
        """One strong-scaling step: broadcast (packed asset) + render share + merge."""
        t, tp_ = pairs[i % len(pairs)]
        fn = pdist.denoise_step_tile_sharded if args.mode.startswith("tiles") else \
            pdist.denoise_step_view_sharded
        return fn(None, intr, c2w, H, W, None, ab, t, tp_, x_in, DV, asset=asset,
                  samples_per_ray=w.samples_per_ray, term_eps=TERM_EPS, engine=args.engine,
                  counters=cnt, timer=timer, p2p=args.mode.endswith("p2p"))

    def step(i, x_in, x_out, cnt=None, timer=None):
        if views_mode and world > 1:
            xp, _, _ = sharded(i, x_in, cnt, timer)
            x_out.copy_(xp)
            return
        t, tp_ = pairs[i % len(pairs)]
        api.dmv3d_render_ddim_step(tp, intr, c2w, H, W, mlp, ab, t, tp_, x_in, None, 0.0, None,
                                   x_prev=x_out, rgb=rgb, alpha=alpha, samples_per_ray=w.samples_per_ray,
                                   term_eps=TERM_EPS, engine=args.engine, counters=cnt, timer=timer)

    # warm-up (untimed), with the kernel's own counters for evaluated samples
    for i in range(args.warmup):
        step(i, xa, xb, counters if i == 0 else None)
        xa, xb = xb, xa
    torch.cuda.synchronize()
    # per-rank kernel counters summed over the ranks (hit / evaluated / tile rows ...)
    cnt_local = counters.cpu().numpy().astype(np.float64)  # this rank's launch (roofline)
    cnt = pdist.sum_over_ranks(cnt_local, dev)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- device-resident timed region: K steps, L2 flushed between steps
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    barrier()
    with ClockSampler(gpu) as clk:
        for k in range(args.steps):
            flush.zero_()
            torch.cuda.nvtx.range_push(f"denoise step {k}")  # NVTX range per loop step
            starts[k].record(stream)
            step(args.warmup + k, xa, xb, timer=kernel_timer)
            ends[k].record(stream)
            torch.cuda.nvtx.range_pop()
            xa, xb = xb, xa
        barrier()
    step_ms = np.array([s.elapsed_time(e) for s, e in zip(starts, ends)])
    total_ms = float(step_ms.sum())
    if world > 1:
        tt = torch.tensor([total_ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms = float(tt.item())
    units_per_step = rays if views_mode else rays * world  # strong vs weak scaling
    value = units_per_step * args.steps / (total_ms / 1e3)
    ms_per_step = total_ms / args.steps

    # ---- sustained clocks: >= sustained_s seconds of the same step, back to back
    sustained = None
    if args.sustained_s > 0:
        n_sus = max(args.steps, int(np.ceil(args.sustained_s * 1e3 / max(ms_per_step, 1e-3))))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        with ClockSampler(gpu) as clk_s:
            e0.record(stream)
            for k in range(n_sus):
                flush.zero_()
                step(k, xa, xb)
                xa, xb = xb, xa
            e1.record(stream)
            barrier()
        sus_ms = pdist.max_over_ranks(e0.elapsed_time(e1), dev)
        sustained = {"steps": n_sus, "seconds": sus_ms / 1e3, "ms_per_step": sus_ms / n_sus,
                     "value": units_per_step * n_sus / (sus_ms / 1e3), "clocks": clk_s.summary()}

    # ---- N > 1: the weak-scaling alternative (one independent asset per rank)
    weak = None
    if world > 1 and views_mode:
        wa = wl.make_workload(wname, asset=rank)
        tpa = torch.from_numpy(wa.triplane).to(dev).to(tdt).contiguous()
        ya, yb = x0.clone(), torch.empty_like(x0)
        for i in range(args.warmup):
            t, tp_ = pairs[i % len(pairs)]
            api.dmv3d_render_ddim_step(tpa, intr, c2w, H, W, mlp, ab, t, tp_, ya, x_prev=yb,
                                       rgb=rgb, alpha=alpha, samples_per_ray=w.samples_per_ray,
                                       term_eps=TERM_EPS, engine=args.engine)
            ya, yb = yb, ya
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for k in range(args.steps):
            flush.zero_()
            t, tp_ = pairs[(args.warmup + k) % len(pairs)]
            api.dmv3d_render_ddim_step(tpa, intr, c2w, H, W, mlp, ab, t, tp_, ya, x_prev=yb,
                                       rgb=rgb, alpha=alpha, samples_per_ray=w.samples_per_ray,
                                       term_eps=TERM_EPS, engine=args.engine)
            ya, yb = yb, ya
        e1.record(stream)
        barrier()
        wk_ms = pdist.max_over_ranks(e0.elapsed_time(e1), dev)
        weak = {"value": rays * world * args.steps / (wk_ms / 1e3), "unit": "rays/s",
                "ms_per_step": wk_ms / args.steps, "scaling": "weak", "assets": world,
                "parallelism": f"asset-sharded x{world}, no data-path collective"}

    # ---- end-to-end through the host-buffer C-ABI entry (pinned host in/out)
    ws = api.Workspace()
    h_tp = tp.cpu().pin_memory()
    h_intr, h_c2w = intr.cpu().pin_memory(), c2w.cpu().pin_memory()
    h_mlp = api.DeviceMLP([x.cpu().pin_memory() for x in mlp.weights],
                          [x.cpu().pin_memory() for x in mlp.biases], w.dtype)
    h_x = [x0.cpu().pin_memory(), torch.empty(x0.shape).pin_memory()]
    h_rgb = torch.empty(rgb.shape).pin_memory()
    h_alpha = torch.empty(alpha.shape).pin_memory()
    h2d = (h_tp.numel() * h_tp.element_size() + h_intr.numel() * 4 + h_c2w.numel() * 4 + h_x[0].numel() * 4
           + sum(x.numel() * x.element_size() for x in h_mlp.weights + h_mlp.biases))
    d2h = h_x[0].numel() * 4 + h_rgb.numel() * 4 + h_alpha.numel() * 4

    if views_mode and world > 1:
        # the public multi-GPU step from host buffers: rank 0 uploads the packed asset and
        # x_t (pinned), broadcasts x_t (the asset broadcast is inside the step), every rank
        # renders its share, rank 0 reads x_{t-1}, rgb and alpha back
        h_flat = asset.flat.cpu().pin_memory()
        xd = torch.empty_like(x0)
        h2d = h_flat.numel() + h_x[0].numel() * 4

        def host_step(i, a, b):
            if rank == 0:
                asset.flat.copy_(h_flat, non_blocking=True)
                xd.copy_(h_x[a], non_blocking=True)
            dist.broadcast(xd, src=0)
            xp, rgb_, alpha_ = sharded(i, xd)
            if rank == 0:
                h_x[b].copy_(xp, non_blocking=True)
                h_rgb.copy_(rgb_, non_blocking=True)
                h_alpha.copy_(alpha_, non_blocking=True)
    else:
        def host_step(i, a, b):
            t, tp_ = pairs[i % len(pairs)]
            api.dmv3d_render_ddim_step_host(ws, h_tp, h_intr, h_c2w, H, W, h_mlp, ab, t, tp_, h_x[a],
                                            h_x[b], h_rgb, h_alpha, samples_per_ray=w.samples_per_ray,
                                            term_eps=TERM_EPS, engine=args.engine, stream=stream)

    for i in range(args.warmup):
        host_step(i, i % 2, (i + 1) % 2)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for k in range(args.steps):
        host_step(args.warmup + k, k % 2, (k + 1) % 2)
        stream.synchronize()  # the step's result is read on the host
    e1.record(stream)
    barrier()
    e2e_ms = e0.elapsed_time(e1)
    if world > 1:
        tt = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms = float(tt.item())
    e2e_value = units_per_step * args.steps / (e2e_ms / 1e3)  # one asset per step (strong)
    ws.close()

    # ---- roofline of the dominant kernel (the fused render kernel: 1 launch / step);
    # per launch on this rank (rank 0), from this rank's own counters
    peaks, peak_src = load_peaks()
    hit_frac = cnt[0] / max(cnt[3], 1)
    eval_samples = cnt[1]  # all ranks, one step
    eval_local = cnt_local[1]
    engine_used = args.engine
    if engine_used == "auto":
        from paper_2605_18052_b200 import _abi
        engine_used = "tcgen05" if _abi.lib() and _tc_available(api, tp, intr, c2w, H, W, mlp) else "simt"
    k_ms, k_launches = kernel_timer.read()  # render-kernel CUDA events, timed region only
    kernel_ms = k_ms / max(k_launches, 1)
    launches_per_step = 2 if engine_used == "tcgen05" else 1  # (pre-projection +) render
    traffic, traffic_note = _ncu_traffic(engine_used)
    if engine_used == "tcgen05":
        flops = eval_local * MLP_FLOPS_PER_SAMPLE
        achieved = flops / (kernel_ms / 1e3) / 1e12
        peak = peaks["bf16_tflops"]
        roof = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_note,
                "peak_source": f"{peak_src} dense bf16 (burst); fp16 operands run at the bf16 rate",
                "kernel": "render_tc_kernel", "kernel_ms": kernel_ms,
                "algorithmic": "27,136 MLP FLOP per evaluated sample x evaluated samples per launch"}
        if "bf16_tflops_sustained" in peaks:
            roof["frac_of_sustained_peak"] = achieved / peaks["bf16_tflops_sustained"]
        dtype = "bf16 storage, fp16 MMA operands, fp32 accumulate"
    else:
        # fp32 CUDA-core engine: MLP + gather FMAs on the FP32 pipe
        flops = eval_local * (MLP_FLOPS_PER_SAMPLE + 2 * 12 * 80)
        achieved = flops / (kernel_ms / 1e3) / 1e12
        sm_mhz = peaks.get("sm_max_mhz", 1965.0)
        peak = 148 * 128 * 2 * sm_mhz * 1e6 / 1e12  # 148 SMs x 128 FP32 lanes x FMA
        roof = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_note,
                "peak_source": "148 SM x 128 FP32 FMA/clk x 2 x sm_max_mhz (DESIGN.md)",
                "kernel": "render_simt_kernel", "kernel_ms": kernel_ms,
                "algorithmic": "(27,136 MLP + 1,920 gather) FLOP per evaluated sample"}
        dtype = "f32 (bf16 storage)"

    # ---- the gather: the triplane is L2-resident, so HBM sees the
    # compulsory bytes (G / the triplane once per step) while the gather itself runs
    # from L2: the tensor-core engine stages each window's texel rows of G (128 B) into
    # shared memory by cp.async and blends them on the tensor cores, the SIMT engine reads
    # 12 C-element texel rows per evaluated sample
    ks = kernel_ms / 1e3
    comp_b = tp.numel() * tp.element_size()
    l2hit, _ = _ncu_traffic(engine_used + "_l2_hit_pct")
    gather = {"bound": "on-chip (L2-resident triplane)", "unit": "GB/s", "hbm_peak": peaks["hbm_gbs"],
              "compulsory_bytes_per_step": comp_b,
              "compulsory_gbs": comp_b / ks / 1e9,
              "compulsory_frac_of_hbm": comp_b / ks / 1e9 / peaks["hbm_gbs"],
              "dram_gbs_ncu": traffic / ks / 1e9 if traffic else None,
              "l2_hit_pct_ncu": l2hit}
    if engine_used == "tcgen05" and cnt_local[4] > 0:
        staged = cnt_local[5] * 128.0  # K columns staged x one 128-B texel row of G each
        gather.update({"l2_to_smem_bytes_per_launch": staged,
                       "l2_to_smem_bytes_per_sample": staged / max(eval_local, 1),
                       "l2_to_smem_gbs": staged / ks / 1e9})
    else:
        req_b = 12 * w.triplane.shape[-1] * tp.element_size()
        gather.update({"requested_bytes_per_sample": req_b,
                       "requested_gbs": eval_local * req_b / ks / 1e9})

    # ---- CPU oracle baseline (rank 0, N = 1 only; bounded sample)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        r_rate, n_rays, secs = oracle_rate(w, args.cpu_budget, threads)
        cpu = {"value": r_rate, "unit": "rays/s", "cores": threads, "kind": "oracle",
               "sample": f"{n_rays} random rays of {args.config} (of {rays}) in {secs:.1f} s; full "
                         f"128-sample march, fp64, no early termination"}
        cpu["cpu_model"] = _cpu_model()
        # the oracle is also timed on one core
        r1, n1, s1 = oracle_rate(w, args.cpu_budget / 3, 1, seed=8)
        cpu["single_core"] = {"value": r1, "unit": "rays/s", "cores": 1,
                              "sample": f"{n1} random rays of {args.config} in {s1:.1f} s"}

    if rank == 0:
        line = {"metric": metric, "value": value, "unit": "rays/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
                "higher_is_better": True, "scaling": "strong" if views_mode else "weak",
                "vs_baseline": None, "dtype": dtype, "data": "synthetic",
                "config": {"workload": workload,
                           "rays_per_step": units_per_step, "assets": 1 if views_mode else world,
                           "engine": engine_used,
                           "l2": "flushed between timed steps (256 MiB write); triplane re-read "
                                 "from HBM each step",
                           "parallelism": (f"16x16 ray tiles interleaved x{world} (packed triplane+MLP broadcast "
                                           + ("+ NVLink peer stores)" if args.mode == "tiles-p2p"
                                              else "+ all-gather of packed tiles)")
                                           if args.mode.startswith("tiles") else
                                           f"view-sharded x{world} (packed triplane+MLP broadcast + "
                                           + ("NVLink peer stores)" if args.mode == "views-p2p"
                                              else "all-gather)")
                                           if views_mode else f"asset-sharded x{world}")},
                "samples_per_s_nominal": value * w.samples_per_ray,
                "samples_per_s_evaluated": eval_samples * args.steps / (total_ms / 1e3),
                "hit_fraction": hit_frac,
                "terminated_fraction_of_hit": cnt[2] / max(cnt[0], 1),
                "evaluated_fraction_of_nominal": eval_samples / (units_per_step * w.samples_per_ray),
                # tensor-core tiles: evaluated samples / MMA rows issued, mean staged K
                "mma_row_occupancy": (eval_samples / cnt[4]) if cnt[4] > 0 else None,
                "mean_blend_k": (cnt[5] / (cnt[4] / 128)) if cnt[4] > 0 else None,
                "roofline": roof, "gather_roofline": gather, "cpu_baseline": cpu,
                "e2e": {"value": e2e_value, "unit": "rays/s", "h2d_bytes_per_step": int(h2d),
                        "d2h_bytes_per_step": int(d2h)},
                "gpu_launches": args.steps * launches_per_step,
                "sustained": sustained, "weak_assets": weak,
                "kernel_ms": kernel_ms, "kernel_share_of_step": kernel_ms / ms_per_step,
                "clocks": clk.summary(), "step_ms_min": float(step_ms.min()),
                "step_ms_median": float(np.median(step_ms))}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def _tc_available(api, tp, intr, c2w, H, W, mlp):
    try:
        api.dmv3d_render_views(tp, intr, c2w, 1, 1, mlp, samples_per_ray=4, engine="tcgen05")
        return True
    except Exception:
        return False


def kernel_source_sha(engine):
    """sha256 (16 hex) of the sources that build the engine's render kernel: a stored ncu
    number is only reported while it describes the kernel being run."""
    import hashlib
    csrc = os.path.join(ROOT, "paper_2605_18052_b200", "csrc")
    files = (["render_tc.cu", "tc_ptx.cuh", "common.cuh"] if engine.startswith("tcgen05")
             else ["render_simt.cu", "simt_common.cuh", "common.cuh"])
    h = hashlib.sha256()
    for f in files:
        with open(os.path.join(csrc, f), "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()[:16]


def _ncu_traffic(engine):
    """(value, note) from profiles/ncu_traffic.json, None if absent or captured from another
    build of the kernel (source sha mismatch)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None, "no ncu capture"
    with open(p) as f:
        d = json.load(f)
    base = engine.split("_")[0]
    ent = d.get(engine)
    if ent is None:
        return None, "no ncu capture"
    want = kernel_source_sha(base)
    got = d.get(base + "_source_sha")
    if got != want:
        return None, f"stale: ncu capture of kernel source {got}, running {want}"
    return ent, f"ncu --set full capture of kernel source {got} ({d.get(base + '_captured', '?')})"


if __name__ == "__main__":
    main()
