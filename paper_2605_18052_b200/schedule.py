"""Host-side diffusion schedule tables fed to the DDIM step (a6).

"add noise according to a cosine schedule" with T = 1000
("t=980/1000 for 50 DDIM denoising steps").  Reading A16: the
improved-DDPM cosine schedule, s = 0.008, beta_j clipped at 0.999, 0-based
alpha_bar_t = prod_{j<=t} (1 - beta_j).  Reading A17: 50 steps, leading
spacing 980, 960, ..., 0; the step after t = 0 is t_prev = -1 (alpha_bar = 1,
fully denoised).
"""
from __future__ import annotations

import numpy as np


def cosine_alpha_bar(T: int = 1000, s: float = 0.008) -> np.ndarray:
    t = np.arange(T + 1, dtype=np.float64)
    f = np.cos(((t / T) + s) / (1.0 + s) * np.pi / 2.0) ** 2
    beta = np.minimum(1.0 - f[1:] / f[:-1], 0.999)
    return np.cumprod(1.0 - beta)


def ddim_timesteps(steps: int = 50, T: int = 1000) -> list[int]:
    stride = T // steps
    return [i * stride for i in reversed(range(steps))]


def ddim_pairs(steps: int = 50, T: int = 1000) -> list[tuple[int, int]]:
    ts = ddim_timesteps(steps, T)
    return list(zip(ts, ts[1:] + [-1]))
