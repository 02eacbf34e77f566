"""Shared test plumbing: move a seeded workload onto the device and into the
oracle's format (bf16 storage is passed to the oracle as its exact fp32 upcast)."""
import numpy as np
import torch

from paper_2605_18052_b200 import api
from paper_2605_18052_b200 import workloads as wl


def dev_workload(w: wl.Workload, device="cuda"):
    dt = torch.bfloat16 if w.dtype == "bf16" else torch.float32
    tp = torch.from_numpy(w.triplane).to(device).to(dt).contiguous()
    intr = torch.from_numpy(w.cameras.intrinsics).to(device)
    c2w = torch.from_numpy(w.cameras.c2w).to(device)
    mlp = api.DeviceMLP.from_host(w.mlp, w.dtype, device)
    return tp, intr, c2w, mlp


def dev_cams(cams: wl.Cameras, device="cuda"):
    return (torch.from_numpy(cams.intrinsics).to(device), torch.from_numpy(cams.c2w).to(device))


def flat_ids(V, H, W, n=None, seed=0):
    total = V * H * W
    if n is None or n >= total:
        return np.arange(total)
    rng = np.random.default_rng(seed)
    ids = rng.choice(total, n, replace=False)
    return np.sort(np.concatenate([ids, [0, total - 1]]))


def pick(img_rgb, img_alpha, ids, H, W):
    """rgb [V,3,H,W], alpha [V,H,W] (numpy) at flat ray ids -> ([n,3], [n])."""
    v = ids // (H * W)
    pix = ids % (H * W)
    i, j = pix // W, pix % W
    return img_rgb[v, :, i, j], img_alpha[v, i, j]


def ddim_tol(alpha_bar, t, t_prev, rgb_tol, x0_scale=2.0):
    """|d x_prev / d rgb| bound for the DDIM map, times the rgb tolerance."""
    abt = alpha_bar[t]
    abp = alpha_bar[t_prev] if t_prev >= 0 else 1.0
    c_eps = np.sqrt(max(0.0, 1 - abp))
    k = abs(x0_scale) * (np.sqrt(abp) + c_eps * np.sqrt(abt) / np.sqrt(1 - abt))
    return k * rgb_tol + 2e-6
