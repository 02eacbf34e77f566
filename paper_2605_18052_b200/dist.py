"""Multi-GPU plumbing: one process per GPU, torch.distributed/NCCL.

The renderer shards with no data-path exchange inside a launch: rays are
independent.  Two partitions are provided, in the priority order of §8e:

* assets (`asset_shard`): a batch of assets (cfg4) is split across ranks and
  every rank runs whole denoising loops on its own assets -- no per-step
  communication at all (weak scaling).
* views (`view_shard` / `denoise_step_view_sharded`): one asset's views are
  split across ranks; per step the owner rank broadcasts the triplane S_t
  (the reconstructor E runs on one rank), every rank renders + DDIM-updates
  its contiguous block of views, and `all_gather_into_tensor` assembles the
  full x_{t-1}, rgb and alpha in place on every rank.  View blocks are whole
  4x4-patch rows, so the gathered result is bitwise equal to one GPU
  rendering all views (pin P12).

* views with P2P outputs (`p2p=True`): the same split, but the outputs live in
  symmetric memory (torch.distributed._symmetric_memory) and the render epilogue
  itself stores every value into all peers' buffers over NVLink (opts.peers of the
  ABI); one device-side barrier replaces the three all-gathers.

* interleaved ray tiles (`denoise_step_tile_sharded`): every rank renders the
  T x T pixel tiles tau = (v ceil(H/T) + i/T) ceil(W/T) + j/T with tau mod P == rank
  of every view (opts.tile_* of the ABI), which spreads AABB misses and early-
  terminated rays evenly; each rank's outputs start at zero, so one all-reduce (sum)
  of the three outputs assembles them (every pixel has exactly one non-zero writer).

The render call is injectable (`render_fn`) so the shard/merge logic is
tested on CPU with gloo and the CPU oracle (tests/test_dist_gloo.py); the
default is libdmv3d's fused step.  The P2P path needs GPUs with peer access; its
kernel side (peer stores) is tested on one GPU with local buffers as peers.
"""
from __future__ import annotations

import math

import torch
import torch.distributed as dist


def view_shard(num_views: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block of views [v0, v1) for `rank`; blocks of ceil(V/P) views,
    the last ranks may get fewer (or none)."""
    per = math.ceil(num_views / world)
    v0 = min(num_views, rank * per)
    return v0, min(num_views, v0 + per)


def asset_shard(num_assets: int, rank: int, world: int) -> list[int]:
    """Assets owned by `rank` (round robin)."""
    return list(range(rank, num_assets, world))


def _gather_views(full: torch.Tensor, v0: int, v1: int, per: int, world: int, group=None):
    """All-gather equal blocks of `per` views into `full` [world*per, ...] in place
    (rank r's block is full[r*per:(r+1)*per]); `full` must have world*per views."""
    rank = dist.get_rank(group)
    mine = full[rank * per:(rank + 1) * per]
    try:
        dist.all_gather_into_tensor(full, mine, group=group)
    except (RuntimeError, NotImplementedError, ValueError):
        # backends without all_gather_into_tensor (e.g. older gloo): list form
        parts = list(full.split(per))  # views into `full`: gathered in place
        dist.all_gather(parts, mine.clone(), group=group)


def peer_pointers(base_ptrs, rank: int, offset_bytes: int) -> list[int]:
    """Addresses of the same element in every other rank's symmetric buffer (bases in
    rank order), in rank order skipping `rank`."""
    return [int(b) + offset_bytes for r, b in enumerate(base_ptrs) if r != rank]


_SYMM = {}


def _symm_outputs(shapes, device, group):
    """Symmetric-memory output tensors (cached per shape set) and their handles."""
    import torch.distributed._symmetric_memory as symm_mem
    key = (tuple(shapes), str(device), id(group))
    if key not in _SYMM:
        name = (group or dist.group.WORLD).group_name
        ts = [symm_mem.empty(*shp, dtype=torch.float32, device=device) for shp in shapes]
        _SYMM[key] = (ts, [symm_mem.rendezvous(t, name) for t in ts])
    return _SYMM[key]


def default_render_fn(triplane, intrinsics, c2w, height, width, mlp, alpha_bar, t, t_prev,
                      x_t, x_prev, rgb, alpha, **opts):
    from . import api
    if x_t is None or x_t.shape[0] == 0:
        api.dmv3d_render_views(triplane, intrinsics, c2w, height, width, mlp, rgb=rgb, alpha=alpha,
                               **opts)
    else:
        api.dmv3d_render_ddim_step(triplane, intrinsics, c2w, height, width, mlp, alpha_bar, t,
                                   t_prev, x_t, x_prev=x_prev, rgb=rgb, alpha=alpha, **opts)


def denoise_step_view_sharded(triplane, intrinsics, c2w, height, width, mlp, alpha_bar, t, t_prev,
                              x_t, ddim_views: int, group=None, src: int = 0,
                              broadcast_triplane: bool = True, render_fn=None, p2p: bool = False,
                              **opts):
    """One denoising step of one asset, views split across the ranks of `group`.

    Every rank passes full-size `intrinsics` [V,4], `c2w` [V,3,4] and `x_t`
    [ddim_views,3,H,W] (only its own block is read).  Returns the full
    (x_prev [ddim_views,3,H,W], rgb [V,3,H,W], alpha [V,H,W]) on every rank.
    `p2p`: outputs in symmetric memory, assembled by the render kernel's peer stores.
    """
    if p2p and dist.get_world_size(group) > 1:
        return _denoise_step_view_sharded_p2p(triplane, intrinsics, c2w, height, width, mlp,
                                              alpha_bar, t, t_prev, x_t, ddim_views, group, src,
                                              broadcast_triplane, render_fn, **opts)
    render_fn = render_fn or default_render_fn
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    V = int(c2w.shape[0])
    per = math.ceil(V / world)
    v0, v1 = view_shard(V, rank, world)
    dev = triplane.device
    if broadcast_triplane and world > 1:
        dist.broadcast(triplane, src=src, group=group)
    # full-size outputs padded to world*per views so every rank's block has the same size
    rgb = torch.empty((world * per, 3, height, width), device=dev, dtype=torch.float32)
    alpha = torch.empty((world * per, height, width), device=dev, dtype=torch.float32)
    xp = torch.empty((world * per, 3, height, width), device=dev, dtype=torch.float32)
    if v1 > v0:
        own_dv = max(0, min(v1, ddim_views) - v0)
        render_fn(triplane, intrinsics[v0:v1].contiguous(), c2w[v0:v1].contiguous(), height, width,
                  mlp, alpha_bar, t, t_prev, x_t[v0:v0 + own_dv] if own_dv else None,
                  xp[v0:v0 + own_dv] if own_dv else None, rgb[v0:v1], alpha[v0:v1], **opts)
    if world > 1:
        _gather_views(rgb, v0, v1, per, world, group)
        _gather_views(alpha, v0, v1, per, world, group)
        _gather_views(xp, v0, v1, per, world, group)
    return xp[:ddim_views], rgb[:V], alpha[:V]


def _denoise_step_view_sharded_p2p(triplane, intrinsics, c2w, height, width, mlp, alpha_bar, t,
                                   t_prev, x_t, ddim_views, group, src, broadcast_triplane,
                                   render_fn, **opts):
    render_fn = render_fn or default_render_fn
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    V = int(c2w.shape[0])
    v0, v1 = view_shard(V, rank, world)
    dev = triplane.device
    if broadcast_triplane:
        dist.broadcast(triplane, src=src, group=group)
    (xp, rgb, alpha), (hx, hr, ha) = _symm_outputs(
        [(max(ddim_views, 1), 3, height, width), (V, 3, height, width), (V, height, width)], dev,
        group)
    if v1 > v0:
        own_dv = max(0, min(v1, ddim_views) - v0)
        HW = height * width
        peers = {"rgb": peer_pointers(hr.buffer_ptrs, rank, v0 * 3 * HW * 4),
                 "alpha": peer_pointers(ha.buffer_ptrs, rank, v0 * HW * 4),
                 "x_prev": peer_pointers(hx.buffer_ptrs, rank, v0 * 3 * HW * 4) if own_dv else []}
        render_fn(triplane, intrinsics[v0:v1].contiguous(), c2w[v0:v1].contiguous(), height, width,
                  mlp, alpha_bar, t, t_prev, x_t[v0:v0 + own_dv] if own_dv else None,
                  xp[v0:v0 + own_dv] if own_dv else None, rgb[v0:v1], alpha[v0:v1], peers=peers,
                  **opts)
    # every rank's peer stores have landed once all ranks pass the device-side barrier
    ha.barrier()
    return xp[:ddim_views], rgb, alpha


def tile_owner(v: int, i: int, j: int, height: int, width: int, tile: int, world: int) -> int:
    """Rank that renders pixel (v, i, j) under the interleaved-tile split."""
    th, tw = -(-height // tile), -(-width // tile)
    return ((v * th + i // tile) * tw + j // tile) % world


def denoise_step_tile_sharded(triplane, intrinsics, c2w, height, width, mlp, alpha_bar, t, t_prev,
                              x_t, ddim_views: int, group=None, src: int = 0,
                              broadcast_triplane: bool = True, render_fn=None, tile: int = 16,
                              p2p: bool = False, **opts):
    """One denoising step of one asset, T x T ray tiles dealt round robin to the ranks.
    Returns the full (x_prev, rgb, alpha) on every rank.  `p2p`: outputs in symmetric
    memory, every rank's render epilogue stores its pixels into all peers' buffers at the
    same offsets (no all-reduce; one device-side barrier)."""
    render_fn = render_fn or default_render_fn
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if p2p and world > 1:
        V = int(c2w.shape[0])
        if broadcast_triplane:
            dist.broadcast(triplane, src=src, group=group)
        (xp, rgb, alpha), (hx, hr, ha) = _symm_outputs(
            [(max(ddim_views, 1), 3, height, width), (V, 3, height, width), (V, height, width)],
            triplane.device, group)
        peers = {"rgb": peer_pointers(hr.buffer_ptrs, rank, 0),
                 "alpha": peer_pointers(ha.buffer_ptrs, rank, 0),
                 "x_prev": peer_pointers(hx.buffer_ptrs, rank, 0) if ddim_views else []}
        render_fn(triplane, intrinsics, c2w, height, width, mlp, alpha_bar, t, t_prev,
                  x_t if ddim_views else None, xp[:ddim_views] if ddim_views else None, rgb, alpha,
                  tiles=(tile, rank, world), peers=peers, **opts)
        ha.barrier()
        return xp[:ddim_views], rgb, alpha
    V = int(c2w.shape[0])
    dev = triplane.device
    if broadcast_triplane and world > 1:
        dist.broadcast(triplane, src=src, group=group)
    HW = height * width
    n_x, n_rgb = ddim_views * 3 * HW, V * 3 * HW
    flat = torch.zeros(n_x + n_rgb + V * HW, device=dev, dtype=torch.float32)  # one collective
    xp = flat[:n_x].view(ddim_views, 3, height, width)
    rgb = flat[n_x:n_x + n_rgb].view(V, 3, height, width)
    alpha = flat[n_x + n_rgb:].view(V, height, width)
    render_fn(triplane, intrinsics, c2w, height, width, mlp, alpha_bar, t, t_prev,
              x_t if ddim_views else None, xp if ddim_views else None, rgb, alpha,
              tiles=(tile, rank, world), **opts)
    if world > 1:
        dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
    return xp, rgb, alpha


def max_over_ranks(value: float, device, group=None) -> float:
    """Device-timed numbers are reported as the max over ranks."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return value
    t = torch.tensor([value], device=device, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
