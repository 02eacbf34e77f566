"""Seeded synthetic inputs shaped like the paper's workloads.

This module is the ONE place shared by the oracle tests and the CUDA path:
it only draws inputs (cameras, triplanes, MLP weights, noise) and holds none
of the method's arithmetic (no ray generation, sampling, gather, MLP
evaluation, compositing or DDIM).  Recipe: DESIGN.md "Input recipe"
(SURVEY.md §8d).

Shapes fixed by PAPER.md:
  * objects scaled to [-1, 1]^3
  * fixed 50 degree FOV
  * 4 inference views uniformly around the object at one pitch,
    elevation 20 deg, azimuths 0/90/180/270
  * 256x256 inputs
  * triplane 3 x 64 x 64 (reading A1); C = 80 (BASELINE.json)
    or 32

Seeds by role: triplane 1 (asset a: 100 + a), MLP 2, cameras 3, x_t 4, z 5.
All arrays are numpy, C-contiguous; float32 unless stated.  bf16 storage is
produced by round-to-nearest-even of the float32 values (``to_bf16_bits``);
``bf16_bits_to_f32`` is the exact upcast both sides read.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

FOV_DEG = 50.0
RADIUS = 2.7
INPUT_ELEVATION_DEG = 20.0
INPUT_AZIMUTHS_DEG = (0.0, 90.0, 180.0, 270.0)
AABB_MIN = (-1.0, -1.0, -1.0)
AABB_MAX = (1.0, 1.0, 1.0)

SEED_TRIPLANE, SEED_MLP, SEED_CAMERAS, SEED_XT, SEED_Z = 1, 2, 3, 4, 5


# --------------------------------------------------------------------------
# bf16 helpers (storage format only)
# --------------------------------------------------------------------------
def to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """float32 -> bf16 bit patterns (uint16), round to nearest even."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    rounding = ((u >> 16) & 1) + 0x7FFF
    out = ((u + rounding) >> 16).astype(np.uint16)
    nan = np.isnan(x)
    if nan.any():
        out[nan] = 0x7FC0
    return out


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    """Exact bf16 -> float32 upcast."""
    return (np.ascontiguousarray(b, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def round_to_bf16(x: np.ndarray) -> np.ndarray:
    """float32 values that are exactly representable in bf16 (RNE)."""
    return bf16_bits_to_f32(to_bf16_bits(x))


def e4m3_values() -> np.ndarray:
    """The 256 OCP FP8 E4M3 code points as float32 (sign | 4-bit exponent, bias 7 | 3-bit
    mantissa; exponent 0 is subnormal; S.1111.111 is NaN, no infinities)."""
    c = np.arange(256)
    sign = np.where(c & 0x80, -1.0, 1.0)
    e, m = (c >> 3) & 0xF, c & 7
    v = np.where(e == 0, m / 8.0 * 2.0 ** -6, (1.0 + m / 8.0) * 2.0 ** (e - 7.0)) * sign
    v[(c & 0x7F) == 0x7F] = np.nan
    return v.astype(np.float32)


def to_e4m3(x: np.ndarray, scale: float = 1.0):
    """x / scale rounded to the nearest E4M3 value (ties to the even code), saturating at
    +-448 -> (codes uint8 [same shape], the stored values scale * e4m3 as float32)."""
    tab = e4m3_values().astype(np.float64)
    pos = np.arange(0, 0x7F)  # finite non-negative codes, increasing values
    y = np.asarray(x, np.float64) / scale
    a = np.minimum(np.abs(y), tab[0x7E])
    i = np.clip(np.searchsorted(tab[pos], a), 1, len(pos) - 1)
    lo, hi = tab[pos[i - 1]], tab[pos[i]]
    take_hi = (a - lo > hi - a) | ((a - lo == hi - a) & (pos[i] % 2 == 0))
    code = np.where(take_hi, pos[i], pos[i - 1]).astype(np.uint8)
    code = np.where((y < 0) & (code != 0), code | 0x80, code).astype(np.uint8)
    vals = (tab[code] * scale).astype(np.float32)
    return code.reshape(np.shape(x)), vals.reshape(np.shape(x))


# --------------------------------------------------------------------------
# cameras
# --------------------------------------------------------------------------
def intrinsics_for(height: int, width: int, fov_deg: float = FOV_DEG) -> np.ndarray:
    """[4] fx, fy, cx, cy in pixels; square pixels, horizontal FOV."""
    f = (width / 2.0) / math.tan(math.radians(fov_deg) / 2.0)
    return np.array([f, f, width / 2.0, height / 2.0], dtype=np.float32)


def look_at_c2w(azimuth_deg: float, elevation_deg: float, radius: float = RADIUS) -> np.ndarray:
    """[3][4] camera-to-world, OpenCV axes (x right, y down, z forward), z-up world,
    camera on a sphere of ``radius`` looking at the origin."""
    az, el = math.radians(azimuth_deg), math.radians(elevation_deg)
    pos = np.array([radius * math.cos(el) * math.cos(az),
                    radius * math.cos(el) * math.sin(az),
                    radius * math.sin(el)], dtype=np.float64)
    fwd = -pos / np.linalg.norm(pos)
    up = np.array([0.0, 0.0, 1.0])
    right = np.cross(fwd, up)
    right /= np.linalg.norm(right)
    down = np.cross(fwd, right)
    m = np.zeros((3, 4), dtype=np.float64)
    m[:, 0], m[:, 1], m[:, 2], m[:, 3] = right, down, fwd, pos
    return m.astype(np.float32)


@dataclasses.dataclass
class Cameras:
    intrinsics: np.ndarray  # [V][4] f32
    c2w: np.ndarray  # [V][3][4] f32
    height: int
    width: int

    @property
    def num_views(self) -> int:
        return int(self.c2w.shape[0])


def input_cameras(height: int, width: int, num_views: int = 4,
                  elevation_deg: float = INPUT_ELEVATION_DEG) -> Cameras:
    """Views uniformly around the object at one pitch."""
    az = [360.0 * k / num_views for k in range(num_views)]
    c2w = np.stack([look_at_c2w(a, elevation_deg) for a in az])
    intr = np.stack([intrinsics_for(height, width)] * num_views)
    return Cameras(np.ascontiguousarray(intr), np.ascontiguousarray(c2w), height, width)


def novel_cameras(height: int, width: int, num_views: int, seed: int = SEED_CAMERAS) -> Cameras:
    """Random novel views: azimuth U[0,360), elevation U[-10,50] (reading A24)."""
    rng = np.random.default_rng(seed)
    az = rng.uniform(0.0, 360.0, num_views)
    el = rng.uniform(-10.0, 50.0, num_views)
    c2w = np.stack([look_at_c2w(a, e) for a, e in zip(az, el)])
    intr = np.stack([intrinsics_for(height, width)] * num_views)
    return Cameras(np.ascontiguousarray(intr), np.ascontiguousarray(c2w), height, width)


def concat_cameras(a: Cameras, b: Cameras) -> Cameras:
    assert a.height == b.height and a.width == b.width
    return Cameras(np.ascontiguousarray(np.concatenate([a.intrinsics, b.intrinsics])),
                   np.ascontiguousarray(np.concatenate([a.c2w, b.c2w])), a.height, a.width)


def axis_camera(height: int, width: int, radius: float = RADIUS) -> Cameras:
    """Camera at (radius, 0, 0) looking at the origin (pin P7)."""
    c2w = look_at_c2w(0.0, 0.0, radius)[None]
    intr = intrinsics_for(height, width)[None]
    return Cameras(np.ascontiguousarray(intr), np.ascontiguousarray(c2w), height, width)


def away_camera(height: int, width: int) -> Cameras:
    """Camera outside the box looking away from it: every ray misses (pin P5)."""
    m = look_at_c2w(0.0, 0.0, RADIUS).astype(np.float64)
    m[:, 0] *= -1.0
    m[:, 2] *= -1.0
    intr = intrinsics_for(height, width)[None]
    return Cameras(np.ascontiguousarray(intr), np.ascontiguousarray(m.astype(np.float32)[None]),
                   height, width)


# --------------------------------------------------------------------------
# triplanes [3][R][R][C], planes XY, XZ, YZ (reading A2)
# --------------------------------------------------------------------------
def texel_world_coords(res: int) -> np.ndarray:
    """World coordinate of texel index 0..R-1 under align-corners (reading A3)."""
    return np.linspace(-1.0, 1.0, res, dtype=np.float64)


def blob_triplane(res: int, channels: int, seed: int = SEED_TRIPLANE, r0: float = 0.9,
                  kappa: float = 10.0) -> np.ndarray:
    """Benchmark default: channel 0 carries a density blob whose mean
    over the planes is kappa*(r0^2 - |p|^2); channels 1.. are N(0, 0.5^2)."""
    rng = np.random.default_rng(seed)
    tp = rng.normal(0.0, 0.5, size=(3, res, res, channels))
    g = texel_world_coords(res)
    col, row = np.meshgrid(g, g, indexing="xy")  # [row][col]
    blob = 1.5 * kappa * ((2.0 / 3.0) * r0 * r0 - col * col - row * row)
    tp[:, :, :, 0] = blob[None]
    return np.ascontiguousarray(tp.astype(np.float32))


def const_triplane(res: int, channels: int, value) -> np.ndarray:
    v = np.broadcast_to(np.asarray(value, dtype=np.float32), (channels,))
    return np.ascontiguousarray(np.broadcast_to(v, (3, res, res, channels)).astype(np.float32))


def linear_triplane(res: int, channels: int, seed: int = SEED_TRIPLANE):
    """F[p][row][col][ch] = a[p,ch]*col + b[p,ch]*row + e[p,ch]; returns (tp, a, b, e)."""
    rng = np.random.default_rng(seed)
    a = rng.uniform(-1, 1, (3, channels))
    b = rng.uniform(-1, 1, (3, channels))
    e = rng.uniform(-1, 1, (3, channels))
    idx = np.arange(res, dtype=np.float64)
    tp = (a[:, None, None, :] * idx[None, None, :, None]
          + b[:, None, None, :] * idx[None, :, None, None] + e[:, None, None, :])
    return np.ascontiguousarray(tp.astype(np.float32)), a, b, e


def random_triplane(res: int, channels: int, seed: int = SEED_TRIPLANE, scale: float = 1.0):
    rng = np.random.default_rng(seed)
    return np.ascontiguousarray(rng.normal(0.0, scale, (3, res, res, channels)).astype(np.float32))


# --------------------------------------------------------------------------
# MLP weights (W_l [out][in], b_l [out]); last layer out = 4 (sigma, r, g, b)
# --------------------------------------------------------------------------
@dataclasses.dataclass
class MLP:
    weights: list  # list of f32 [out][in]
    biases: list  # list of f32 [out]
    hidden_act: int = 0  # 0 relu, 1 silu, 2 softplus
    density_shift: float = 0.0
    rgb_widen_eps: float = 0.0

    @property
    def num_layers(self) -> int:
        return len(self.weights)

    @property
    def in_dim(self) -> int:
        return int(self.weights[0].shape[1])

    @property
    def hidden(self) -> int:
        return int(self.weights[0].shape[0]) if self.num_layers > 1 else 4


def _torch_default_linear(rng, out_dim, in_dim):
    bound = 1.0 / math.sqrt(in_dim)
    return rng.uniform(-bound, bound, (out_dim, in_dim)), rng.uniform(-bound, bound, out_dim)


def random_mlp(in_dim: int, hidden: int, num_layers: int, seed: int = SEED_MLP) -> MLP:
    rng = np.random.default_rng(seed)
    ws, bs = [], []
    d = in_dim
    for l in range(num_layers):
        o = 4 if l == num_layers - 1 else hidden
        w, b = _torch_default_linear(rng, o, d)
        ws.append(np.ascontiguousarray(w.astype(np.float32)))
        bs.append(np.ascontiguousarray(b.astype(np.float32)))
        d = o
    return MLP(ws, bs)


def blob_mlp(in_dim: int, hidden: int, num_layers: int, seed: int = SEED_MLP,
             sigma_gain: float = 20.0, sigma_bias: float = -6.0) -> MLP:
    """Benchmark default: hidden unit 0 of every layer forwards
    max(channel 0, 0); the sigma row is [gain, 0, ...] with bias -6."""
    m = random_mlp(in_dim, hidden, num_layers, seed)
    ws = [w.astype(np.float64) for w in m.weights]
    bs = [b.astype(np.float64) for b in m.biases]
    for l in range(num_layers - 1):
        ws[l][0, :] = 0.0
        ws[l][:, 0] = 0.0
        ws[l][0, 0] = 1.0
        bs[l][0] = 0.0
    last = ws[-1]
    last[:, 0] = 0.0
    last[0, :] = 0.0
    last[0, 0] = sigma_gain
    bs[-1][0] = sigma_bias
    return MLP([np.ascontiguousarray(w.astype(np.float32)) for w in ws],
               [np.ascontiguousarray(b.astype(np.float32)) for b in bs])


def bf16_mlp(m: MLP) -> MLP:
    """Weights rounded to bf16-representable float32 (biases stay f32)."""
    return MLP([round_to_bf16(w) for w in m.weights], [b.copy() for b in m.biases],
               m.hidden_act, m.density_shift, m.rgb_widen_eps)


# --------------------------------------------------------------------------
# diffusion noise
# --------------------------------------------------------------------------
def gaussian(shape, seed: int) -> np.ndarray:
    return np.ascontiguousarray(np.random.default_rng(seed).standard_normal(shape).astype(np.float32))


# --------------------------------------------------------------------------
# named configurations (BASELINE.json configs)
# --------------------------------------------------------------------------
@dataclasses.dataclass
class Workload:
    name: str
    triplane: np.ndarray  # f32 [3][R][R][C] (bf16-representable when dtype == "bf16")
    cameras: Cameras
    mlp: MLP
    samples_per_ray: int
    dtype: str  # "f32" or "bf16"
    ddim_views: int = 0  # first ddim_views views get the DDIM epilogue
    bg: tuple = (1.0, 1.0, 1.0)

    @property
    def res(self):
        return int(self.triplane.shape[1])

    @property
    def channels(self):
        return int(self.triplane.shape[3])

    @property
    def num_rays(self):
        return self.cameras.num_views * self.cameras.height * self.cameras.width


def make_workload(name: str, asset: int | None = None) -> Workload:
    tseed = SEED_TRIPLANE if asset is None else 100 + asset
    if name == "cfg1":
        tp = blob_triplane(8, 4, tseed, kappa=4.0)
        return Workload(name, tp, input_cameras(16, 16, 1), blob_mlp(4, 16, 2), 16, "f32")
    if name in ("cfg2", "cfg2_bf16"):
        dt = "bf16" if name.endswith("bf16") else "f32"
        tp = blob_triplane(64, 80, tseed)
        m = blob_mlp(80, 64, 4)
        if dt == "bf16":
            tp, m = round_to_bf16(tp), bf16_mlp(m)
        return Workload(name, tp, input_cameras(128, 128, 4), m, 128, dt)
    if name in ("cfg3", "cfg3_c32", "cfg3_l2", "cfg3_f32"):
        C = 32 if name == "cfg3_c32" else 80
        L = 2 if name == "cfg3_l2" else 4
        dt = "f32" if name == "cfg3_f32" else "bf16"
        tp = blob_triplane(64, C, tseed)
        m = blob_mlp(C, 64, L)
        if dt == "bf16":
            tp, m = round_to_bf16(tp), bf16_mlp(m)
        cams = concat_cameras(input_cameras(256, 256, 4), novel_cameras(256, 256, 4))
        return Workload(name, tp, cams, m, 128, dt, ddim_views=4)
    raise KeyError(name)
