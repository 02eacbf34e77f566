"""Python binding of libdmv3d (same names as the C ABI, argument marshalling only).

PyTorch supplies device memory and the current CUDA stream; every step of the
path (rays, samples, gather, MLP, compositing, DDIM) runs in libdmv3d's
kernels.  There is no fallback: a missing library or a non-OK status raises.
"""
from __future__ import annotations

import ctypes as ct
import dataclasses

import numpy as np
import torch

from . import _abi

_DT = {"f32": _abi.F32, "bf16": _abi.BF16}
_TORCH_DT = {"f32": torch.float32, "bf16": torch.bfloat16}
_ENGINE = {"auto": _abi.ENGINE_AUTO, "simt": _abi.ENGINE_SIMT, "tcgen05": _abi.ENGINE_TCGEN05}
_AGG = {"mean": _abi.AGG_MEAN, "sum": _abi.AGG_SUM, "concat": _abi.AGG_CONCAT}
# texel addressing (reading A3; row f4): grid_sample align_corners=True + border, or
# align_corners=False + zero padding
_SMODE = {"align_corners": _abi.SAMPLE_ALIGN_CORNERS, "halfpixel_zeros": _abi.SAMPLE_HALFPIXEL_ZEROS}


def _ptr(t):
    return None if t is None else ct.c_void_p(t.data_ptr())


def _stream(device=None):
    return ct.c_void_p(torch.cuda.current_stream(device).cuda_stream)


@dataclasses.dataclass
class DeviceMLP:
    """Shared MLP on the device: weights W_l [out][in] (f32 or bf16), biases f32."""
    weights: list
    biases: list
    dtype: str
    hidden_act: int = 0
    density_shift: float = 0.0
    rgb_widen_eps: float = 0.0

    @classmethod
    def from_host(cls, m, dtype: str = "f32", device="cuda"):
        ws = [torch.from_numpy(np.ascontiguousarray(w)).to(device=device, dtype=_TORCH_DT[dtype])
              for w in m.weights]
        bs = [torch.from_numpy(np.ascontiguousarray(b, dtype=np.float32)).to(device) for b in m.biases]
        return cls(ws, bs, dtype, m.hidden_act, m.density_shift, m.rgb_widen_eps)

    def struct(self, keep):
        L = len(self.weights)
        warr = (ct.c_void_p * L)(*[w.data_ptr() for w in self.weights])
        barr = (ct.c_void_p * L)(*[b.data_ptr() for b in self.biases])
        keep += [warr, barr]
        hidden = int(self.weights[0].shape[0]) if L > 1 else 4
        return _abi.MLP(L, int(self.weights[0].shape[1]), hidden, _DT[self.dtype],
                        ct.cast(warr, ct.POINTER(ct.c_void_p)), ct.cast(barr, ct.POINTER(ct.c_void_p)),
                        self.hidden_act, self.density_shift, self.rgb_widen_eps)


def triplane_struct(tp: torch.Tensor, aabb_min=(-1.0, -1.0, -1.0), aabb_max=(1.0, 1.0, 1.0),
                    sample_mode="align_corners", fp8_scale=1.0):
    """`tp` float32 / bfloat16 / float8_e4m3fn (value = fp8_scale * e4m3, TCGEN05 only);
    [3,R,R,C], or [A,3,R,R,C] for the batched entry points."""
    if tp.dim() == 5:
        tp = tp[0]
    assert tp.dim() == 4 and tp.shape[0] == 3 and tp.shape[1] == tp.shape[2] and tp.is_contiguous()
    dt = {torch.float32: _abi.F32, torch.bfloat16: _abi.BF16,
          torch.float8_e4m3fn: _abi.FP8_E4M3}[tp.dtype]
    return _abi.Triplane(int(tp.shape[1]), int(tp.shape[3]), dt, tp.data_ptr(),
                         (ct.c_float * 3)(*aabb_min), (ct.c_float * 3)(*aabb_max),
                         _SMODE[sample_mode], fp8_scale)


def cameras_struct(intrinsics: torch.Tensor, c2w: torch.Tensor, height: int, width: int):
    """[V,4] / [V,3,4], or [A,V,4] / [A,V,3,4] for the batched entry points (V per asset)."""
    assert intrinsics.dtype == torch.float32 and c2w.dtype == torch.float32
    assert intrinsics.is_contiguous() and c2w.is_contiguous()
    return _abi.Cameras(int(c2w.shape[-3]), height, width, intrinsics.data_ptr(), c2w.data_ptr())


def opts_struct(samples_per_ray=128, agg="mean", jitter=False, seed=0, bg=(1.0, 1.0, 1.0),
                term_eps=0.0, ray_range=None, engine="auto", counters=None, workspace=None,
                timer=None, plucker=None, peers=None, fwd=None, tiles=None):
    """`peers`: optional dict with "rgb" / "alpha" / "x_prev" lists of device addresses
    (ints, 0 = skip) laid out like the corresponding outputs (P2P copies, see the ABI).
    `fwd`: (rgb, alpha) of the forward render, for the backward (opts.fwd_rgb / fwd_alpha).
    `tiles`: (tile_size, rank, count): interleaved ray tiles, only this rank's are rendered."""
    b, e = (-1, -1) if ray_range is None else ray_range
    ws_ptr = None if workspace is None else workspace.data_ptr()
    ws_len = 0 if workspace is None else workspace.numel() * workspace.element_size()
    o = _abi.RenderOpts(samples_per_ray, _AGG[agg], 1 if jitter else 0, seed,
                        (ct.c_float * 3)(*bg), term_eps, b, e, _ENGINE[engine],
                        None if counters is None else counters.data_ptr(), ws_ptr, ws_len,
                        None if timer is None else timer.handle,
                        None if plucker is None else plucker.data_ptr())
    if fwd is not None:
        o.fwd_rgb, o.fwd_alpha = fwd[0].data_ptr(), fwd[1].data_ptr()
    if tiles is not None:
        o.tile_size, o.tile_rank, o.tile_count = (int(x) for x in tiles)
    if peers:
        n = max(len(peers.get(k) or []) for k in ("rgb", "alpha", "x_prev"))
        arrs = {}
        for k in ("rgb", "alpha", "x_prev"):
            vals = list(peers.get(k) or []) + [0] * n
            arrs[k] = (ct.c_void_p * n)(*[v or None for v in vals[:n]])
        o.num_peers = n
        o.peer_rgb = ct.cast(arrs["rgb"], ct.c_void_p)
        o.peer_alpha = ct.cast(arrs["alpha"], ct.c_void_p)
        o.peer_x_prev = ct.cast(arrs["x_prev"], ct.c_void_p)
        o._keep = arrs  # the arrays must outlive the call
    return o


def dmv3d_render_backward(triplane, intrinsics, c2w, height, width, mlp: "DeviceMLP", grad_rgb,
                          grad_alpha=None, aabb_min=(-1.0,) * 3, aabb_max=(1.0,) * 3, **opts):
    """Gradients of <grad_rgb, rgb> + <grad_alpha, alpha> w.r.t. the triplane and the MLP
    (row f1) -> (d_triplane [3,R,R,C] f32, [dW_l] f32, [db_l] f32).  engine="tcgen05" runs
    the tensor-core backward (bf16 storage; a workspace is attached), otherwise fp32 SIMT."""
    dev = triplane.device
    dF = torch.zeros(triplane.shape, device=dev, dtype=torch.float32)
    dW = [torch.zeros(w.shape, device=dev, dtype=torch.float32) for w in mlp.weights]
    db = [torch.zeros(b.shape, device=dev, dtype=torch.float32) for b in mlp.biases]
    keep = []
    t = triplane_struct(triplane, aabb_min, aabb_max, opts.pop("sample_mode", "align_corners"),
                        fp8_scale=opts.pop("fp8_scale", 1.0))
    c = cameras_struct(intrinsics, c2w, height, width)
    m = mlp.struct(keep)
    if opts.get("engine") == "tcgen05" and "workspace" not in opts:  # tensor-core backward
        opts["workspace"] = workspace_for(t, m, dev, torch.cuda.current_stream(dev))
    o = opts_struct(**opts)
    L = len(dW)
    dWp = (ct.c_void_p * L)(*[x.data_ptr() for x in dW])
    dbp = (ct.c_void_p * L)(*[x.data_ptr() for x in db])
    _abi.check(_abi.lib().dmv3d_render_backward(ct.byref(t), ct.byref(c), ct.byref(m), ct.byref(o),
                                                _ptr(grad_rgb), _ptr(grad_alpha), _ptr(dF),
                                                ct.cast(dWp, ct.POINTER(ct.c_void_p)),
                                                ct.cast(dbp, ct.POINTER(ct.c_void_p)),
                                                _stream(dev)))
    return dF, dW, db


def dmv3d_density_grid(triplane, mlp: "DeviceMLP", grid_res, want_rgb=True, agg="mean",
                       aabb_min=(-1.0,) * 3, aabb_max=(1.0,) * 3, timer=None, engine="auto",
                       sample_mode="align_corners", fp8_scale=1.0):
    """sigma [G,G,G] (+ rgb [3,G,G,G]) of the decoder on the box grid."""
    G = int(grid_res)
    dev = triplane.device
    sigma = torch.empty((G, G, G), device=dev, dtype=torch.float32)
    rgb = torch.empty((3, G, G, G), device=dev, dtype=torch.float32) if want_rgb else None
    keep = []
    t = triplane_struct(triplane, aabb_min, aabb_max, sample_mode, fp8_scale)
    m = mlp.struct(keep)
    ws = workspace_for(t, m, dev, torch.cuda.current_stream(dev))
    o = opts_struct(agg=agg, engine=engine, workspace=ws, timer=timer)
    _abi.check(_abi.lib().dmv3d_density_grid(ct.byref(t), ct.byref(m), ct.byref(o), G, _ptr(sigma),
                                             _ptr(rgb), _stream(dev)))
    return sigma, rgb


def dmv3d_plucker_rays(intrinsics, c2w, height, width, out=None, ray_range=None):
    """Plucker ray map (o x d, d) [V,6,H,W] of the renderer's rays."""
    V = int(c2w.shape[0])
    if out is None:
        out = torch.empty((V, 6, height, width), device=c2w.device, dtype=torch.float32)
    c = cameras_struct(intrinsics, c2w, height, width)
    o = opts_struct(samples_per_ray=1, ray_range=ray_range)
    _abi.check(_abi.lib().dmv3d_plucker_rays(ct.byref(c), ct.byref(o), _ptr(out),
                                             _stream(c2w.device)))
    return out


def tiles_per_rank(num_views, height, width, tile, world):
    """Blocks per rank of the tile-packed layout: ceil(tiles / world)."""
    ntiles = num_views * -(-height // tile) * -(-width // tile)
    return -(-ntiles // world)


def dmv3d_tiles_pack(intrinsics, c2w, height, width, tile, rank, world, rgb=None, alpha=None,
                     x_prev=None, packed_rgb=None, packed_alpha=None, packed_x_prev=None,
                     ddim_views=0):
    """Copy rank `rank`'s interleaved tiles from image-layout outputs into its packed
    blocks (rgb [nmax,3,T,T], alpha [nmax,T,T], x_prev [nmax,3,T,T])."""
    c = cameras_struct(intrinsics, c2w, height, width)
    _abi.check(_abi.lib().dmv3d_tiles_pack(ct.byref(c), int(tile), int(rank), int(world),
                                           int(ddim_views), _ptr(rgb), _ptr(alpha), _ptr(x_prev),
                                           _ptr(packed_rgb), _ptr(packed_alpha),
                                           _ptr(packed_x_prev), _stream(c2w.device)))


def dmv3d_tiles_unpack(intrinsics, c2w, height, width, tile, world, packed_rgb=None,
                       packed_alpha=None, packed_x_prev=None, rgb=None, alpha=None, x_prev=None,
                       ddim_views=0):
    """Scatter `world` ranks' gathered tile-packed outputs ([world * tiles_per_rank, ...])
    into image-layout rgb [V,3,H,W], alpha [V,H,W], x_prev [ddim_views,3,H,W]."""
    c = cameras_struct(intrinsics, c2w, height, width)
    _abi.check(_abi.lib().dmv3d_tiles_unpack(ct.byref(c), int(tile), int(world), int(ddim_views),
                                             _ptr(packed_rgb), _ptr(packed_alpha),
                                             _ptr(packed_x_prev), _ptr(rgb), _ptr(alpha),
                                             _ptr(x_prev), _stream(c2w.device)))


class Timer:
    """dmv3d_timer: CUDA events the library records around each render kernel."""

    def __init__(self):
        self.handle = ct.c_void_p()
        _abi.check(_abi.lib().dmv3d_timer_create(ct.byref(self.handle)))

    def reset(self):
        _abi.check(_abi.lib().dmv3d_timer_reset(self.handle))

    def read(self):
        """(total device ms, number of bracketed launches) since the last reset."""
        ms, n = ct.c_double(), ct.c_int64()
        _abi.check(_abi.lib().dmv3d_timer_read(self.handle, ct.byref(ms), ct.byref(n)))
        return ms.value, n.value

    def close(self):
        if self.handle:
            _abi.lib().dmv3d_timer_destroy(self.handle)
            self.handle = ct.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_WS_CACHE = {}


def workspace_for(triplane_s, mlp_s, device, stream=None, assets=1):
    """Device scratch for the tensor-core engine (dmv3d_workspace_bytes[_batched]), cached
    per (device, stream): calls that share a workspace must be ordered on one stream."""
    n = int(_abi.lib().dmv3d_workspace_bytes_batched(ct.byref(triplane_s), ct.byref(mlp_s),
                                                     int(assets)))
    if n == 0 or device.type != "cuda":
        return None
    key = (device.index, None if stream is None else stream.cuda_stream)
    buf = _WS_CACHE.get(key)
    if buf is None or buf.numel() < n:
        buf = torch.empty(n, dtype=torch.uint8, device=device)
        _WS_CACHE[key] = buf
    return buf


RANGE_G_OVERFLOW, RANGE_ACT_OVERFLOW = 1, 2


def dmv3d_range_flags(workspace=None, device=None):
    """fp16 range flags of the last tensor-core call that used `workspace` (default: this
    module's cached workspace of `device` / the current stream): bit 0 = the projected
    triplane left +-65504, bit 1 = an fp16 activation overflowed (non-finite head
    output).  Non-zero: that call's outputs hold inf / NaN.  Synchronises the stream."""
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if workspace is None:
        workspace = _WS_CACHE.get((dev.index, torch.cuda.current_stream(dev).cuda_stream))
        if workspace is None:
            return 0
    out = ct.c_uint32()
    _abi.check(_abi.lib().dmv3d_range_flags(ct.c_void_p(workspace.data_ptr()), ct.byref(out),
                                            _stream(dev)))
    return int(out.value)


def dmv3d_select_engine(triplane, mlp: "DeviceMLP", assets=1, aabb_min=(-1.0,) * 3,
                        aabb_max=(1.0,) * 3, **opts):
    """The engine a render / DDIM call with these arguments runs: "tcgen05" or "simt"."""
    dev = triplane.device
    keep = []
    tt = triplane_struct(triplane, aabb_min, aabb_max, opts.pop("sample_mode", "align_corners"),
                         fp8_scale=opts.pop("fp8_scale", 1.0))
    m = mlp.struct(keep)
    if "workspace" not in opts:
        opts["workspace"] = workspace_for(tt, m, dev, torch.cuda.current_stream(dev), assets=assets)
    o = opts_struct(**opts)
    e = ct.c_int32()
    _abi.check(_abi.lib().dmv3d_select_engine(ct.byref(tt), ct.byref(m), ct.byref(o), int(assets),
                                              ct.byref(e)))
    return {1: "simt", 2: "tcgen05"}[e.value]


def ddim_struct(alpha_bar: np.ndarray, t: int, t_prev: int, eta: float, keep_mask, ddim_views,
                keep, x0_scale=2.0, x0_shift=-1.0, noise_seed=None, skip_kept_views=False):
    ab = np.ascontiguousarray(alpha_bar, dtype=np.float64)
    keep.append(ab)
    km = None
    if keep_mask is not None:
        km = np.ascontiguousarray(keep_mask, dtype=np.uint8)
        keep.append(km)
    return _abi.DdimParams(ab.ctypes.data_as(ct.POINTER(ct.c_double)), len(ab), t, t_prev, eta,
                           x0_scale, x0_shift,
                           km.ctypes.data_as(ct.POINTER(ct.c_uint8)) if km is not None else None,
                           ddim_views, 0 if noise_seed is None else 1,
                           0 if noise_seed is None else int(noise_seed), 1 if skip_kept_views else 0)


# ------------------------------------------------------------------- entry points
def dmv3d_render_views(triplane, intrinsics, c2w, height, width, mlp: DeviceMLP, rgb=None,
                       alpha=None, aabb_min=(-1.0,) * 3, aabb_max=(1.0,) * 3, **opts):
    """R(S, c) for every view -> rgb [V,3,H,W], alpha [V,H,W]."""
    V = int(c2w.shape[0])
    dev = triplane.device
    if rgb is None:
        rgb = torch.empty((V, 3, height, width), device=dev, dtype=torch.float32)
    if alpha is None:
        alpha = torch.empty((V, height, width), device=dev, dtype=torch.float32)
    keep = []
    t = triplane_struct(triplane, aabb_min, aabb_max, opts.pop("sample_mode", "align_corners"),
                        fp8_scale=opts.pop("fp8_scale", 1.0))
    c = cameras_struct(intrinsics, c2w, height, width)
    m = mlp.struct(keep)
    if "workspace" not in opts:
        opts["workspace"] = workspace_for(t, m, dev, torch.cuda.current_stream(dev))
    o = opts_struct(**opts)
    _abi.check(_abi.lib().dmv3d_render_views(ct.byref(t), ct.byref(c), ct.byref(m), ct.byref(o),
                                             _ptr(rgb), _ptr(alpha), _stream(dev)))
    return rgb, alpha


def dmv3d_ddim_step(alpha_bar, t, t_prev, x_t, x0_rgb, z=None, eta=0.0, keep_mask=None,
                    x_prev=None, x0_scale=2.0, x0_shift=-1.0, noise_seed=None):
    """Standalone DDIM x0 -> x_{t-1} over [V,3,H,W]; z = None with
    noise_seed set draws the fresh noise in the kernel (row f4)."""
    V, _, H, W = x_t.shape
    if x_prev is None:
        x_prev = torch.empty_like(x_t)
    keep = []
    d = ddim_struct(alpha_bar, t, t_prev, eta, keep_mask, V, keep, x0_scale, x0_shift, noise_seed)
    _abi.check(_abi.lib().dmv3d_ddim_step(ct.byref(d), V, H, W, _ptr(x_t), _ptr(x0_rgb), _ptr(z),
                                          _ptr(x_prev), _stream(x_t.device)))
    return x_prev


def dmv3d_render_ddim_step(triplane, intrinsics, c2w, height, width, mlp: DeviceMLP, alpha_bar,
                           t, t_prev, x_t, z=None, eta=0.0, keep_mask=None, x_prev=None,
                           rgb=None, alpha=None, want_rgb=True, want_alpha=True,
                           aabb_min=(-1.0,) * 3, aabb_max=(1.0,) * 3, x0_scale=2.0,
                           x0_shift=-1.0, noise_seed=None, skip_kept_views=False, **opts):
    """Fused step: render all views; views [0, x_t.shape[0]) also get x_{t-1}.  With
    want_rgb = want_alpha = False only those views are rendered; skip_kept_views: views
    with keep_mask set are not rendered (x_{t-1} = x_t, their rgb/alpha untouched)."""
    V = int(c2w.shape[0])
    dv = int(x_t.shape[0])
    dev = triplane.device
    if x_prev is None:
        x_prev = torch.empty_like(x_t)
    if rgb is None and want_rgb:
        rgb = torch.empty((V, 3, height, width), device=dev, dtype=torch.float32)
    if alpha is None and want_alpha:
        alpha = torch.empty((V, height, width), device=dev, dtype=torch.float32)
    keep = []
    tt = triplane_struct(triplane, aabb_min, aabb_max, opts.pop("sample_mode", "align_corners"),
                        fp8_scale=opts.pop("fp8_scale", 1.0))
    c = cameras_struct(intrinsics, c2w, height, width)
    m = mlp.struct(keep)
    if "workspace" not in opts:
        opts["workspace"] = workspace_for(tt, m, dev, torch.cuda.current_stream(dev))
    o = opts_struct(**opts)
    d = ddim_struct(alpha_bar, t, t_prev, eta, keep_mask, dv, keep, x0_scale, x0_shift, noise_seed,
                    skip_kept_views)
    _abi.check(_abi.lib().dmv3d_render_ddim_step(ct.byref(tt), ct.byref(c), ct.byref(m),
                                                 ct.byref(o), ct.byref(d), _ptr(x_t), _ptr(z),
                                                 _ptr(x_prev), _ptr(rgb), _ptr(alpha),
                                                 _stream(dev)))
    return x_prev, rgb, alpha


def dmv3d_render_ddim_step_batched(triplane, intrinsics, c2w, height, width, mlp: DeviceMLP,
                                   alpha_bar, t, t_prev, x_t, z=None, eta=0.0, keep_mask=None,
                                   x_prev=None, rgb=None, alpha=None, want_rgb=True,
                                   want_alpha=True, aabb_min=(-1.0,) * 3, aabb_max=(1.0,) * 3,
                                   x0_scale=2.0, x0_shift=-1.0, noise_seed=None,
                                   skip_kept_views=False, **opts):
    """Batched fused step (one launch for A assets sharing the MLP, cfg4): triplane
    [A,3,R,R,C], intrinsics [A,V,4], c2w [A,V,3,4], x_t [A,DV,3,H,W] ->
    (x_prev [A,DV,3,H,W], rgb [A,V,3,H,W], alpha [A,V,H,W])."""
    A, V = int(c2w.shape[0]), int(c2w.shape[1])
    dv = int(x_t.shape[1])
    dev = triplane.device
    assert triplane.dim() == 5 and triplane.shape[0] == A and x_t.shape[0] == A
    if x_prev is None:
        x_prev = torch.empty_like(x_t)
    if rgb is None and want_rgb:
        rgb = torch.empty((A, V, 3, height, width), device=dev, dtype=torch.float32)
    if alpha is None and want_alpha:
        alpha = torch.empty((A, V, height, width), device=dev, dtype=torch.float32)
    keep = []
    tt = triplane_struct(triplane, aabb_min, aabb_max, opts.pop("sample_mode", "align_corners"),
                         fp8_scale=opts.pop("fp8_scale", 1.0))
    c = cameras_struct(intrinsics, c2w, height, width)
    m = mlp.struct(keep)
    if "workspace" not in opts:
        opts["workspace"] = workspace_for(tt, m, dev, torch.cuda.current_stream(dev), assets=A)
    o = opts_struct(**opts)
    d = ddim_struct(alpha_bar, t, t_prev, eta, keep_mask, dv, keep, x0_scale, x0_shift, noise_seed,
                    skip_kept_views)
    _abi.check(_abi.lib().dmv3d_render_ddim_step_batched(ct.byref(tt), A, ct.byref(c), ct.byref(m),
                                                         ct.byref(o), ct.byref(d), _ptr(x_t),
                                                         _ptr(z), _ptr(x_prev), _ptr(rgb),
                                                         _ptr(alpha), _stream(dev)))
    return x_prev, rgb, alpha


def dmv3d_render_views_batched(triplane, intrinsics, c2w, height, width, mlp: DeviceMLP,
                               rgb=None, alpha=None, aabb_min=(-1.0,) * 3, aabb_max=(1.0,) * 3,
                               **opts):
    """Batched R(S, c): triplane [A,3,R,R,C], cameras [A,V,...] -> rgb [A,V,3,H,W],
    alpha [A,V,H,W]."""
    A, V = int(c2w.shape[0]), int(c2w.shape[1])
    dev = triplane.device
    if rgb is None:
        rgb = torch.empty((A, V, 3, height, width), device=dev, dtype=torch.float32)
    if alpha is None:
        alpha = torch.empty((A, V, height, width), device=dev, dtype=torch.float32)
    keep = []
    tt = triplane_struct(triplane, aabb_min, aabb_max, opts.pop("sample_mode", "align_corners"),
                         fp8_scale=opts.pop("fp8_scale", 1.0))
    c = cameras_struct(intrinsics, c2w, height, width)
    m = mlp.struct(keep)
    if "workspace" not in opts:
        opts["workspace"] = workspace_for(tt, m, dev, torch.cuda.current_stream(dev), assets=A)
    o = opts_struct(**opts)
    _abi.check(_abi.lib().dmv3d_render_views_batched(ct.byref(tt), A, ct.byref(c), ct.byref(m),
                                                     ct.byref(o), _ptr(rgb), _ptr(alpha),
                                                     _stream(dev)))
    return rgb, alpha


class Workspace:
    """Owner of the library's grow-only device buffers for the host-buffer entry."""

    def __init__(self):
        self.handle = ct.c_void_p()
        _abi.check(_abi.lib().dmv3d_workspace_create(ct.byref(self.handle)))

    def range_flags(self):
        """fp16 range flags of the last host-buffer step (see dmv3d_range_flags)."""
        out = ct.c_uint32()
        _abi.check(_abi.lib().dmv3d_workspace_range_flags(self.handle, ct.byref(out)))
        return int(out.value)

    def close(self):
        if self.handle:
            _abi.lib().dmv3d_workspace_destroy(self.handle)
            self.handle = ct.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def dmv3d_render_ddim_step_host(ws: Workspace, triplane, intrinsics, c2w, height, width, mlp,
                                alpha_bar, t, t_prev, x_t, x_prev, rgb=None, alpha=None, z=None,
                                eta=0.0, keep_mask=None, stream=None, **opts):
    """Host-buffer step: every tensor is a (pinned) CPU tensor; copies in/out are inside
    the library call, on `stream` (default: torch's current stream)."""
    keep = []
    tt = triplane_struct(triplane, sample_mode=opts.pop("sample_mode", "align_corners"),
                        fp8_scale=opts.pop("fp8_scale", 1.0))
    c = cameras_struct(intrinsics, c2w, height, width)
    m = mlp.struct(keep)
    o = opts_struct(**opts)
    d = ddim_struct(alpha_bar, t, t_prev, eta, keep_mask, int(x_t.shape[0]), keep)
    st = ct.c_void_p(stream.cuda_stream) if stream is not None else _stream()
    _abi.check(_abi.lib().dmv3d_render_ddim_step_host(ws.handle, ct.byref(tt), ct.byref(c),
                                                      ct.byref(m), ct.byref(o), ct.byref(d),
                                                      _ptr(x_t), _ptr(z), _ptr(x_prev),
                                                      _ptr(rgb), _ptr(alpha), st))
    return x_prev, rgb, alpha


# ------------------------------------------------------------ stage-level (debug)
def dmv3d_debug_ray_geometry(intrinsics, c2w, height, width, aabb_min=(-1.0,) * 3,
                             aabb_max=(1.0,) * 3, ray_range=None):
    V = int(c2w.shape[0])
    n = V * height * width if ray_range is None else ray_range[1] - ray_range[0]
    dev = c2w.device
    o_d = torch.empty((n, 6), device=dev)
    tn_tf = torch.empty((n, 2), device=dev)
    hit = torch.empty((n,), device=dev, dtype=torch.uint8)
    c = cameras_struct(intrinsics, c2w, height, width)
    o = opts_struct(ray_range=ray_range)
    lo, hi = (ct.c_float * 3)(*aabb_min), (ct.c_float * 3)(*aabb_max)
    _abi.check(_abi.lib().dmv3d_debug_ray_geometry(ct.byref(c), lo, hi, ct.byref(o), _ptr(o_d),
                                                   _ptr(tn_tf), _ptr(hit), _stream(dev)))
    return o_d, tn_tf, hit


def dmv3d_debug_sample_points(intrinsics, c2w, height, width, res, samples_per_ray,
                              aabb_min=(-1.0,) * 3, aabb_max=(1.0,) * 3, ray_range=None,
                              jitter=False, seed=0, sample_mode="align_corners"):
    V = int(c2w.shape[0])
    n = V * height * width if ray_range is None else ray_range[1] - ray_range[0]
    N = samples_per_ray
    dev = c2w.device
    t_k = torch.empty((n, N), device=dev)
    pts = torch.empty((n, N, 3), device=dev)
    texel = torch.empty((n, N, 3, 2), device=dev, dtype=torch.int32)
    frac = torch.empty((n, N, 3, 2), device=dev)
    c = cameras_struct(intrinsics, c2w, height, width)
    o = opts_struct(samples_per_ray=N, ray_range=ray_range, jitter=jitter, seed=seed)
    grid = _abi.Triplane(int(res), 4, _abi.F32, None, (ct.c_float * 3)(*aabb_min),
                         (ct.c_float * 3)(*aabb_max), _SMODE[sample_mode])
    _abi.check(_abi.lib().dmv3d_debug_sample_points(ct.byref(c), ct.byref(grid), ct.byref(o),
                                                    _ptr(t_k), _ptr(pts), _ptr(texel),
                                                    _ptr(frac), _stream(dev)))
    return t_k, pts, texel, frac


def dmv3d_debug_sample_features(triplane, points, agg="mean", sample_mode="align_corners"):
    n = int(points.shape[0])
    k = int(triplane.shape[3]) * (3 if agg == "concat" else 1)
    feats = torch.empty((n, k), device=triplane.device)
    t = triplane_struct(triplane, sample_mode=sample_mode)
    _abi.check(_abi.lib().dmv3d_debug_sample_features(ct.byref(t), _AGG[agg], n, _ptr(points),
                                                      _ptr(feats), _stream(triplane.device)))
    return feats


def dmv3d_debug_decode(triplane, mlp: DeviceMLP, points, agg="mean", sample_mode="align_corners"):
    n = int(points.shape[0])
    out = torch.empty((n, 4), device=triplane.device)
    keep = []
    t = triplane_struct(triplane, sample_mode=sample_mode)
    m = mlp.struct(keep)
    _abi.check(_abi.lib().dmv3d_debug_decode(ct.byref(t), ct.byref(m), _AGG[agg], n, _ptr(points),
                                             _ptr(out), _stream(triplane.device)))
    return out


# short aliases (the C names above are the canonical ones)
render_views = dmv3d_render_views
ddim_step = dmv3d_ddim_step
render_ddim_step = dmv3d_render_ddim_step
