"""ctypes mirror of include/dmv3d.h (argument marshalling only).

Loads the in-tree libdmv3d.so; raises if it is missing -- there is no CPU or
PyTorch fallback for any step of the path.
"""
from __future__ import annotations

import ctypes as ct
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# DMV3D_LIB selects an instrumented in-tree build (tools/phases.py); default: the product
LIB_PATH = os.environ.get("DMV3D_LIB") or os.path.join(HERE, "libdmv3d.so")

OK, ERR_INVALID_ARG, ERR_UNSUPPORTED, ERR_CUDA, ERR_ALIGNMENT = 0, 1, 2, 3, 4
F32, BF16, FP8_E4M3 = 0, 1, 2
AGG_MEAN, AGG_SUM, AGG_CONCAT = 0, 1, 2
SAMPLE_ALIGN_CORNERS, SAMPLE_HALFPIXEL_ZEROS = 0, 1
ACT_RELU, ACT_SILU, ACT_SOFTPLUS = 0, 1, 2
ENGINE_AUTO, ENGINE_SIMT, ENGINE_TCGEN05 = 0, 1, 2

EXPORTED = [
    "dmv3d_render_views", "dmv3d_ddim_step", "dmv3d_render_ddim_step", "dmv3d_last_error",
    "dmv3d_version", "dmv3d_workspace_create", "dmv3d_workspace_destroy",
    "dmv3d_render_ddim_step_host", "dmv3d_debug_ray_geometry", "dmv3d_debug_sample_points",
    "dmv3d_debug_sample_features", "dmv3d_debug_decode", "dmv3d_workspace_bytes",
    "dmv3d_timer_create", "dmv3d_timer_destroy", "dmv3d_timer_reset", "dmv3d_timer_read",
    "dmv3d_plucker_rays", "dmv3d_density_grid", "dmv3d_render_backward",
    "dmv3d_render_views_batched", "dmv3d_render_ddim_step_batched", "dmv3d_workspace_bytes_batched",
    "dmv3d_range_flags", "dmv3d_workspace_range_flags", "dmv3d_select_engine",
    "dmv3d_tiles_pack", "dmv3d_tiles_unpack",
]


class Cameras(ct.Structure):
    _fields_ = [("num_views", ct.c_int32), ("height", ct.c_int32), ("width", ct.c_int32),
                ("intrinsics", ct.c_void_p), ("c2w", ct.c_void_p)]


class Triplane(ct.Structure):
    _fields_ = [("res", ct.c_int32), ("channels", ct.c_int32), ("dtype", ct.c_int32),
                ("data", ct.c_void_p), ("aabb_min", ct.c_float * 3), ("aabb_max", ct.c_float * 3),
                ("sample_mode", ct.c_int32), ("fp8_scale", ct.c_float)]


class MLP(ct.Structure):
    _fields_ = [("num_layers", ct.c_int32), ("in_dim", ct.c_int32), ("hidden", ct.c_int32),
                ("dtype", ct.c_int32), ("weights", ct.POINTER(ct.c_void_p)),
                ("biases", ct.POINTER(ct.c_void_p)), ("hidden_act", ct.c_int32),
                ("density_shift", ct.c_float), ("rgb_widen_eps", ct.c_float)]


class RenderOpts(ct.Structure):
    _fields_ = [("samples_per_ray", ct.c_int32), ("agg", ct.c_int32), ("jitter", ct.c_int32),
                ("seed", ct.c_uint64), ("bg_rgb", ct.c_float * 3), ("term_eps", ct.c_float),
                ("ray_begin", ct.c_int64), ("ray_end", ct.c_int64), ("engine", ct.c_int32),
                ("counters", ct.c_void_p), ("workspace", ct.c_void_p),
                ("workspace_bytes", ct.c_uint64), ("timer", ct.c_void_p),
                ("plucker", ct.c_void_p), ("num_peers", ct.c_int32),
                ("peer_rgb", ct.c_void_p), ("peer_alpha", ct.c_void_p),
                ("peer_x_prev", ct.c_void_p), ("tile_size", ct.c_int32), ("tile_rank", ct.c_int32),
                ("tile_count", ct.c_int32), ("fwd_rgb", ct.c_void_p), ("fwd_alpha", ct.c_void_p)]


class DdimParams(ct.Structure):
    _fields_ = [("alpha_bar", ct.POINTER(ct.c_double)), ("T", ct.c_int32), ("t", ct.c_int32),
                ("t_prev", ct.c_int32), ("eta", ct.c_float), ("x0_scale", ct.c_float),
                ("x0_shift", ct.c_float), ("keep_mask", ct.POINTER(ct.c_uint8)),
                ("ddim_views", ct.c_int32), ("noise_in_kernel", ct.c_int32),
                ("noise_seed", ct.c_uint64), ("skip_kept_views", ct.c_int32)]


class DMV3DError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"dmv3d status {status}: {msg}")
        self.status = status


_lib = None


def lib() -> ct.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                              "(python -m paper_2605_18052_b200.build); there is no fallback")
        L = ct.CDLL(LIB_PATH)
        P = ct.POINTER
        L.dmv3d_last_error.restype = ct.c_char_p
        L.dmv3d_version.restype = ct.c_char_p
        L.dmv3d_render_views.argtypes = [P(Triplane), P(Cameras), P(MLP), P(RenderOpts),
                                         ct.c_void_p, ct.c_void_p, ct.c_void_p]
        L.dmv3d_ddim_step.argtypes = [P(DdimParams), ct.c_int32, ct.c_int32, ct.c_int32,
                                      ct.c_void_p, ct.c_void_p, ct.c_void_p, ct.c_void_p,
                                      ct.c_void_p]
        L.dmv3d_render_ddim_step.argtypes = [P(Triplane), P(Cameras), P(MLP), P(RenderOpts),
                                             P(DdimParams), ct.c_void_p, ct.c_void_p,
                                             ct.c_void_p, ct.c_void_p, ct.c_void_p, ct.c_void_p]
        L.dmv3d_render_views_batched.argtypes = [P(Triplane), ct.c_int32, P(Cameras), P(MLP),
                                                 P(RenderOpts), ct.c_void_p, ct.c_void_p,
                                                 ct.c_void_p]
        L.dmv3d_render_ddim_step_batched.argtypes = [P(Triplane), ct.c_int32, P(Cameras), P(MLP),
                                                     P(RenderOpts), P(DdimParams), ct.c_void_p,
                                                     ct.c_void_p, ct.c_void_p, ct.c_void_p,
                                                     ct.c_void_p, ct.c_void_p]
        L.dmv3d_workspace_bytes_batched.argtypes = [P(Triplane), P(MLP), ct.c_int32]
        L.dmv3d_workspace_bytes_batched.restype = ct.c_uint64
        L.dmv3d_workspace_create.argtypes = [P(ct.c_void_p)]
        L.dmv3d_workspace_destroy.argtypes = [ct.c_void_p]
        L.dmv3d_render_ddim_step_host.argtypes = [ct.c_void_p, P(Triplane), P(Cameras), P(MLP),
                                                  P(RenderOpts), P(DdimParams), ct.c_void_p,
                                                  ct.c_void_p, ct.c_void_p, ct.c_void_p,
                                                  ct.c_void_p, ct.c_void_p]
        L.dmv3d_debug_ray_geometry.argtypes = [P(Cameras), P(ct.c_float), P(ct.c_float),
                                               P(RenderOpts), ct.c_void_p, ct.c_void_p,
                                               ct.c_void_p, ct.c_void_p]
        L.dmv3d_debug_sample_points.argtypes = [P(Cameras), P(Triplane), P(RenderOpts), ct.c_void_p,
                                                ct.c_void_p, ct.c_void_p, ct.c_void_p,
                                                ct.c_void_p]
        L.dmv3d_debug_sample_features.argtypes = [P(Triplane), ct.c_int32, ct.c_int64,
                                                  ct.c_void_p, ct.c_void_p, ct.c_void_p]
        L.dmv3d_debug_decode.argtypes = [P(Triplane), P(MLP), ct.c_int32, ct.c_int64,
                                         ct.c_void_p, ct.c_void_p, ct.c_void_p]
        L.dmv3d_plucker_rays.argtypes = [P(Cameras), P(RenderOpts), ct.c_void_p, ct.c_void_p]
        L.dmv3d_render_backward.argtypes = [P(Triplane), P(Cameras), P(MLP), P(RenderOpts),
                                            ct.c_void_p, ct.c_void_p, ct.c_void_p,
                                            P(ct.c_void_p), P(ct.c_void_p), ct.c_void_p]
        L.dmv3d_density_grid.argtypes = [P(Triplane), P(MLP), P(RenderOpts), ct.c_int32,
                                         ct.c_void_p, ct.c_void_p, ct.c_void_p]
        L.dmv3d_timer_create.argtypes = [P(ct.c_void_p)]
        L.dmv3d_timer_destroy.argtypes = [ct.c_void_p]
        L.dmv3d_timer_reset.argtypes = [ct.c_void_p]
        L.dmv3d_timer_read.argtypes = [ct.c_void_p, P(ct.c_double), P(ct.c_int64)]
        L.dmv3d_range_flags.argtypes = [ct.c_void_p, P(ct.c_uint32), ct.c_void_p]
        L.dmv3d_tiles_unpack.argtypes = [P(Cameras), ct.c_int32, ct.c_int32, ct.c_int32, ct.c_void_p,
                                         ct.c_void_p, ct.c_void_p, ct.c_void_p, ct.c_void_p,
                                         ct.c_void_p, ct.c_void_p]
        L.dmv3d_tiles_pack.argtypes = [P(Cameras), ct.c_int32, ct.c_int32, ct.c_int32, ct.c_int32,
                                       ct.c_void_p, ct.c_void_p, ct.c_void_p, ct.c_void_p,
                                       ct.c_void_p, ct.c_void_p, ct.c_void_p]
        L.dmv3d_workspace_range_flags.argtypes = [ct.c_void_p, P(ct.c_uint32)]
        L.dmv3d_select_engine.argtypes = [P(Triplane), P(MLP), P(RenderOpts), ct.c_int32,
                                          P(ct.c_int32)]
        L.dmv3d_workspace_bytes.argtypes = [P(Triplane), P(MLP)]
        L.dmv3d_workspace_bytes.restype = ct.c_uint64
        for name in EXPORTED:
            if name not in ("dmv3d_last_error", "dmv3d_version", "dmv3d_workspace_bytes",
                            "dmv3d_workspace_bytes_batched"):
                getattr(L, name).restype = ct.c_int
        _lib = L
    return _lib


def check(status: int) -> None:
    if status != OK:
        raise DMV3DError(status, lib().dmv3d_last_error().decode())
