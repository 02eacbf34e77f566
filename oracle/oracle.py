"""ctypes wrapper of liboracle.so (oracle/dmv3d_oracle.c).  TEST INFRASTRUCTURE ONLY.

Functions mirror the paper's definitions (see dmv3d_oracle.h for citations).
Inputs are numpy arrays; bf16 inputs must be passed as their exact float32
upcast (paper_2605_18052_b200.workloads.bf16_bits_to_f32), so the oracle
measures compute precision, not input quantisation.
"""
from __future__ import annotations

import ctypes as ct
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "dmv3d_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

AGG_MEAN, AGG_SUM, AGG_CONCAT = 0, 1, 2
SAMPLE_ALIGN_CORNERS, SAMPLE_HALFPIXEL_ZEROS = 0, 1


def build(force: bool = False) -> str:
    """Compile liboracle.so: -O2 -fopenmp -ffp-contract=off, no fast-math."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "dmv3d_oracle.h"))):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fopenmp", "-ffp-contract=off",
                               "-fno-fast-math", "-fPIC", "-shared", "-D_GNU_SOURCE",
                               "-o", _LIB, _SRC, "-lm"])
    return _LIB


class _Triplane(ct.Structure):
    _fields_ = [("res", ct.c_int32), ("channels", ct.c_int32), ("data", ct.POINTER(ct.c_double)),
                ("aabb_min", ct.c_float * 3), ("aabb_max", ct.c_float * 3),
                ("sample_mode", ct.c_int32)]


class _MLP(ct.Structure):
    _fields_ = [("num_layers", ct.c_int32), ("in_dim", ct.c_int32), ("hidden", ct.c_int32),
                ("weights", ct.POINTER(ct.POINTER(ct.c_double))),
                ("biases", ct.POINTER(ct.POINTER(ct.c_double))),
                ("hidden_act", ct.c_int32), ("density_shift", ct.c_double),
                ("rgb_widen_eps", ct.c_double)]


class _Cameras(ct.Structure):
    _fields_ = [("num_views", ct.c_int32), ("height", ct.c_int32), ("width", ct.c_int32),
                ("intrinsics", ct.POINTER(ct.c_float)), ("c2w", ct.POINTER(ct.c_float))]


class _Opts(ct.Structure):
    _fields_ = [("samples_per_ray", ct.c_int32), ("agg", ct.c_int32), ("jitter", ct.c_int32),
                ("seed", ct.c_uint64), ("bg", ct.c_double * 3)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ct.CDLL(build())
        P = ct.POINTER
        f32p, f64p = P(ct.c_float), P(ct.c_double)
        _lib.orc_cosine_alpha_bar.argtypes = [ct.c_int32, ct.c_double, f64p]
        _lib.orc_ray_geometry.argtypes = [P(_Cameras), f32p, f32p, ct.c_int64, f32p, f32p, f32p,
                                          f32p, P(ct.c_int32)]
        _lib.orc_jitter.argtypes = [ct.c_uint64, ct.c_uint64]
        _lib.orc_jitter.restype = ct.c_float
        _lib.orc_sample_point.argtypes = [f32p, f32p, ct.c_float, ct.c_float, ct.c_int32,
                                          ct.c_int32, ct.c_int32, ct.c_uint64, ct.c_int64, f32p,
                                          f32p]
        _lib.orc_texel_coord.argtypes = [ct.c_float, ct.c_float, ct.c_float, ct.c_int32,
                                         P(ct.c_int32), f32p]
        _lib.orc_point_features.argtypes = [P(_Triplane), ct.c_int32, f32p, f64p]
        _lib.orc_mlp_decode.argtypes = [P(_MLP), f64p, f64p, f64p]
        _lib.orc_decode_point.argtypes = [P(_Triplane), P(_MLP), ct.c_int32, f32p, f64p]
        _lib.orc_render_ray.argtypes = [P(_Triplane), P(_Cameras), P(_MLP), P(_Opts), ct.c_int64,
                                        f64p, f64p]
        _lib.orc_render_rays.argtypes = [P(_Triplane), P(_Cameras), P(_MLP), P(_Opts),
                                         ct.c_int64, P(ct.c_int64), f64p, f64p, ct.c_int32]
        _lib.orc_render_views.argtypes = [P(_Triplane), P(_Cameras), P(_MLP), P(_Opts), f64p,
                                          f64p, ct.c_int32]
        _lib.orc_ddim_step.argtypes = [f64p, ct.c_int32, ct.c_int32, ct.c_int32, ct.c_double,
                                       ct.c_double, ct.c_double, ct.c_int32, ct.c_int32,
                                       ct.c_int32, f64p, f64p, f64p, P(ct.c_uint8), f64p]
    return _lib


def _fp(a):
    return a.ctypes.data_as(ct.POINTER(ct.c_float))


def _dp(a):
    return a.ctypes.data_as(ct.POINTER(ct.c_double))


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


class _Keep:
    """Holds numpy buffers alive while ctypes structs point into them."""

    def __init__(self):
        self.refs = []

    def __call__(self, a):
        self.refs.append(a)
        return a


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _triplane(tp, keep, aabb_min=(-1, -1, -1), aabb_max=(1, 1, 1), sample_mode=0):
    tp = keep(_f64(tp))  # fp32 / bf16-valued inputs upcast exactly
    s = _Triplane(tp.shape[1], tp.shape[3], _dp(tp), (ct.c_float * 3)(*aabb_min),
                  (ct.c_float * 3)(*aabb_max), sample_mode)
    return s


def _mlp(m, keep):
    ws = [keep(_f64(w)) for w in m.weights]
    bs = [keep(_f64(b)) for b in m.biases]
    L = len(ws)
    warr = keep((ct.POINTER(ct.c_double) * L)(*[_dp(w) for w in ws]))
    barr = keep((ct.POINTER(ct.c_double) * L)(*[_dp(b) for b in bs]))
    hidden = ws[0].shape[0] if L > 1 else 4
    return _MLP(L, ws[0].shape[1], hidden, warr, barr, m.hidden_act, m.density_shift,
                m.rgb_widen_eps)


def _cams(c, keep):
    intr = keep(_f32(c.intrinsics))
    c2w = keep(_f32(c.c2w))
    return _Cameras(c2w.shape[0], c.height, c.width, _fp(intr), _fp(c2w))


def _opts(N, agg=AGG_MEAN, jitter=0, seed=0, bg=(1.0, 1.0, 1.0)):
    return _Opts(N, agg, jitter, seed, (ct.c_double * 3)(*bg))


# ------------------------------------------------------------------ API
def cosine_alpha_bar(T: int = 1000, s: float = 0.008) -> np.ndarray:
    out = np.zeros(T, dtype=np.float64)
    lib().orc_cosine_alpha_bar(T, s, _dp(out))
    return out


def ray_geometry(cams, ray_ids, aabb_min=(-1, -1, -1), aabb_max=(1, 1, 1)):
    """fp32 geometry for ray ids -> (o [n,3], d [n,3], t_near [n], t_far [n], hit [n])."""
    keep = _Keep()
    c = _cams(cams, keep)
    lo = keep(_f32(aabb_min))
    hi = keep(_f32(aabb_max))
    ray_ids = np.asarray(ray_ids, dtype=np.int64)
    n = len(ray_ids)
    o = np.zeros((n, 3), np.float32)
    d = np.zeros((n, 3), np.float32)
    tn = np.zeros(n, np.float32)
    tf = np.zeros(n, np.float32)
    hit = np.zeros(n, np.int32)
    L = lib()
    for q, r in enumerate(ray_ids):
        oo, dd = np.zeros(3, np.float32), np.zeros(3, np.float32)
        a, b = ct.c_float(), ct.c_float()
        h = ct.c_int32()
        L.orc_ray_geometry(ct.byref(c), _fp(lo), _fp(hi), int(r), _fp(oo), _fp(dd), ct.byref(a),
                           ct.byref(b), ct.byref(h))
        o[q], d[q], tn[q], tf[q], hit[q] = oo, dd, a.value, b.value, h.value
    return o, d, tn, tf, hit


def plucker(cams, ray_ids):
    """Plucker rays (o x d, d) -> [n, 6] fp32."""
    keep = _Keep()
    c = _cams(cams, keep)
    L = lib()
    L.orc_plucker.argtypes = [ct.POINTER(_Cameras), ct.c_int64, ct.POINTER(ct.c_float)]
    out = np.zeros((len(ray_ids), 6), np.float32)
    for q, r in enumerate(np.asarray(ray_ids, dtype=np.int64)):
        row = np.zeros(6, np.float32)
        L.orc_plucker(ct.byref(c), int(r), _fp(row))
        out[q] = row
    return out


def render_backward(tp, cams, m, N, grad_rgb, grad_alpha=None, agg=AGG_MEAN, jitter=0, seed=0,
                    bg=(1.0, 1.0, 1.0), sample_mode=0):
    """Gradients of L = sum(grad_rgb * rgb) + sum(grad_alpha * alpha) w.r.t. the triplane
    and the MLP (row f1) -> (dF [3,R,R,C], [dW_l], [db_l]), fp64."""
    keep = _Keep()
    t = _triplane(tp, keep, sample_mode=sample_mode)
    mm = _mlp(m, keep)
    c = _cams(cams, keep)
    o = _opts(N, agg, jitter, seed, bg)
    dF = np.zeros(np.shape(tp), np.float64)
    dW = [np.zeros(np.shape(w), np.float64) for w in m.weights]
    db = [np.zeros(np.shape(b), np.float64) for b in m.biases]
    L = len(dW)
    dWp = (ct.POINTER(ct.c_double) * L)(*[_dp(x) for x in dW])
    dbp = (ct.POINTER(ct.c_double) * L)(*[_dp(x) for x in db])
    gr = _f64(grad_rgb)
    ga = _f64(grad_alpha) if grad_alpha is not None else None
    Lb = lib()
    Lb.orc_render_backward.argtypes = [ct.POINTER(_Triplane), ct.POINTER(_Cameras),
                                       ct.POINTER(_MLP), ct.POINTER(_Opts),
                                       ct.POINTER(ct.c_double), ct.POINTER(ct.c_double),
                                       ct.POINTER(ct.c_double),
                                       ct.POINTER(ct.POINTER(ct.c_double)),
                                       ct.POINTER(ct.POINTER(ct.c_double))]
    Lb.orc_render_backward(ct.byref(t), ct.byref(c), ct.byref(mm), ct.byref(o), _dp(gr),
                           _dp(ga) if ga is not None else None, _dp(dF), dWp, dbp)
    return dF, dW, db


def grid_points(G, aabb_min=(-1, -1, -1), aabb_max=(1, 1, 1)):
    """[G^3, 3] fp32 grid points of the density grid (x fastest)."""
    L = lib()
    L.orc_grid_point.argtypes = [ct.POINTER(ct.c_float), ct.POINTER(ct.c_float), ct.c_int32,
                                 ct.c_int64, ct.POINTER(ct.c_float)]
    lo, hi = _f32(aabb_min), _f32(aabb_max)
    out = np.zeros((G ** 3, 3), np.float32)
    for q in range(G ** 3):
        row = np.zeros(3, np.float32)
        L.orc_grid_point(_fp(lo), _fp(hi), G, q, _fp(row))
        out[q] = row
    return out


def density_grid(tp, m, G, agg=AGG_MEAN, threads=0, aabb_min=(-1, -1, -1), aabb_max=(1, 1, 1),
                 sample_mode=0):
    """sigma [G,G,G] and rgb [3,G,G,G] (fp64) on the density grid (row f3)."""
    keep = _Keep()
    t = _triplane(tp, keep, aabb_min, aabb_max, sample_mode)
    mm = _mlp(m, keep)
    L = lib()
    L.orc_density_grid.argtypes = [ct.POINTER(_Triplane), ct.POINTER(_MLP), ct.c_int32, ct.c_int32,
                                   ct.POINTER(ct.c_double), ct.POINTER(ct.c_double), ct.c_int32]
    sigma = np.zeros((G, G, G), np.float64)
    rgb = np.zeros((3, G, G, G), np.float64)
    L.orc_density_grid(ct.byref(t), ct.byref(mm), agg, G, _dp(sigma), _dp(rgb), threads)
    return sigma, rgb


def noise(seed: int, n: int) -> np.ndarray:
    """In-kernel DDIM noise z for elements 0..n-1 (row f4), fp64."""
    L = lib()
    L.orc_noise.argtypes = [ct.c_uint64, ct.c_uint64]
    L.orc_noise.restype = ct.c_double
    return np.array([L.orc_noise(seed, e) for e in range(n)], np.float64)


def jitter(seed: int, sample_id: int) -> float:
    return lib().orc_jitter(seed, sample_id)


def sample_point(o, d, t_near, t_far, N, k, jit=0, seed=0, r=0):
    o, d = _f32(o), _f32(d)
    p = np.zeros(3, np.float32)
    t = ct.c_float()
    lib().orc_sample_point(_fp(o), _fp(d), float(t_near), float(t_far), N, k, jit, seed, r,
                           ct.byref(t), _fp(p))
    return np.float32(t.value), p


def texel_coord(q, lo, hi, R, sample_mode=0):
    i0 = ct.c_int32()
    f = ct.c_float()
    fn = lib().orc_texel_coord_halfpixel if sample_mode == 1 else lib().orc_texel_coord
    fn.argtypes = [ct.c_float, ct.c_float, ct.c_float, ct.c_int32, ct.POINTER(ct.c_int32),
                   ct.POINTER(ct.c_float)]
    fn(float(q), float(lo), float(hi), R, ct.byref(i0), ct.byref(f))
    return i0.value, np.float32(f.value)


def point_features(tp, points, agg=AGG_MEAN, sample_mode=0):
    keep = _Keep()
    t = _triplane(tp, keep, sample_mode=sample_mode)
    pts = _f32(points).reshape(-1, 3)
    K = tp.shape[3] * (3 if agg == AGG_CONCAT else 1)
    out = np.zeros((len(pts), K), np.float64)
    for q in range(len(pts)):
        p = np.ascontiguousarray(pts[q])
        row = np.zeros(K, np.float64)
        lib().orc_point_features(ct.byref(t), agg, _fp(p), _dp(row))
        out[q] = row
    return out


def mlp_decode(m, h0):
    keep = _Keep()
    mm = _mlp(m, keep)
    h0 = np.ascontiguousarray(np.atleast_2d(h0), dtype=np.float64)
    out = np.zeros((len(h0), 4), np.float64)
    for q in range(len(h0)):
        s = ct.c_double()
        rgb = np.zeros(3, np.float64)
        lib().orc_mlp_decode(ct.byref(mm), _dp(np.ascontiguousarray(h0[q])), ct.byref(s), _dp(rgb))
        out[q, 0] = s.value
        out[q, 1:] = rgb
    return out


def decode_points(tp, m, points, agg=AGG_MEAN, sample_mode=0):
    keep = _Keep()
    t = _triplane(tp, keep, sample_mode=sample_mode)
    mm = _mlp(m, keep)
    pts = _f32(points).reshape(-1, 3)
    out = np.zeros((len(pts), 4), np.float64)
    for q in range(len(pts)):
        row = np.zeros(4, np.float64)
        lib().orc_decode_point(ct.byref(t), ct.byref(mm), agg, _fp(np.ascontiguousarray(pts[q])),
                               _dp(row))
        out[q] = row
    return out


def render_rays(tp, cams, m, N, ray_ids, agg=AGG_MEAN, jitter=0, seed=0, bg=(1.0, 1.0, 1.0),
                threads=0, aabb_min=(-1, -1, -1), aabb_max=(1, 1, 1), sample_mode=0):
    """Render selected ray ids -> rgb [n,3], alpha [n] (fp64)."""
    keep = _Keep()
    t = _triplane(tp, keep, aabb_min, aabb_max, sample_mode)
    mm = _mlp(m, keep)
    c = _cams(cams, keep)
    o = _opts(N, agg, jitter, seed, bg)
    ids = np.ascontiguousarray(ray_ids, dtype=np.int64)
    rgb = np.zeros((len(ids), 3), np.float64)
    alpha = np.zeros(len(ids), np.float64)
    lib().orc_render_rays(ct.byref(t), ct.byref(c), ct.byref(mm), ct.byref(o), len(ids),
                          ids.ctypes.data_as(ct.POINTER(ct.c_int64)), _dp(rgb), _dp(alpha),
                          threads)
    return rgb, alpha


def render_views(tp, cams, m, N, agg=AGG_MEAN, jitter=0, seed=0, bg=(1.0, 1.0, 1.0), threads=0,
                 aabb_min=(-1, -1, -1), aabb_max=(1, 1, 1), sample_mode=0):
    """Render all views -> rgb [V,3,H,W], alpha [V,H,W] (fp64)."""
    keep = _Keep()
    t = _triplane(tp, keep, aabb_min, aabb_max, sample_mode)
    mm = _mlp(m, keep)
    c = _cams(cams, keep)
    o = _opts(N, agg, jitter, seed, bg)
    V, H, W = cams.num_views, cams.height, cams.width
    rgb = np.zeros((V, 3, H, W), np.float64)
    alpha = np.zeros((V, H, W), np.float64)
    lib().orc_render_views(ct.byref(t), ct.byref(c), ct.byref(mm), ct.byref(o), _dp(rgb),
                           _dp(alpha), threads)
    return rgb, alpha


def ddim_step(alpha_bar, t, t_prev, x_t, x0_rgb, z=None, eta=0.0, keep_mask=None,
              x0_scale=2.0, x0_shift=-1.0):
    """x_{t-1} from x_t and the rendered x0 image, all [V,3,H,W] (fp64)."""
    ab = np.ascontiguousarray(alpha_bar, dtype=np.float64)
    x_t = np.ascontiguousarray(x_t, dtype=np.float64)
    x0 = np.ascontiguousarray(x0_rgb, dtype=np.float64)
    V, _, H, W = x_t.shape
    zz = np.ascontiguousarray(z, dtype=np.float64) if z is not None else None
    km = np.ascontiguousarray(keep_mask, dtype=np.uint8) if keep_mask is not None else None
    out = np.zeros_like(x_t)
    lib().orc_ddim_step(_dp(ab), len(ab), t, t_prev, eta, x0_scale, x0_shift, V, H, W, _dp(x_t),
                        _dp(x0), _dp(zz) if zz is not None else None,
                        km.ctypes.data_as(ct.POINTER(ct.c_uint8)) if km is not None else None,
                        _dp(out))
    return out
