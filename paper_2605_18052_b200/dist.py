"""Multi-GPU plumbing: one process per GPU, torch.distributed/NCCL.

The renderer shards with no data-path exchange inside a launch: rays are independent
and a denoising step needs one exchange (every step renders the
views from the current triplane, whose owner is the reconstructor's rank).  Partitions,
in the priority order of §8e:

* assets (`asset_shard`): a batch of assets (cfg4) is split across ranks; every rank
  runs whole denoising loops on its own assets (batched launches) -- no per-step
  communication at all (weak scaling).
* views (`denoise_step_view_sharded`): one asset's views in contiguous blocks per
  rank.  Every rank passes the FULL camera set and x_t and renders the ray range of its
  views, so view ids, keep_mask bits, x_t / x_{t-1} offsets and in-kernel noise
  counters are the global ones; the outputs live in buffers padded to world * per views
  and one coalesced all-gather (rgb, alpha, x_{t-1}) assembles them in place.  Whole
  views are whole 4x4-patch rows, so the result is bitwise the one-GPU step (P12).
* interleaved ray tiles (`denoise_step_tile_sharded`): the T x T tiles
  tau = (v ceil(H/T) + i/T) ceil(W/T) + j/T with tau mod P == rank (opts.tile_*),
  which spreads AABB misses and early-terminated rays evenly.  Each rank packs its
  tiles block by block (`dmv3d_tiles_pack`); one coalesced all-gather of the packed
  blocks and `dmv3d_tiles_unpack` assemble the images (`packed=False`: zeroed full-size
  outputs merged by one all-reduce, ~2x the bytes), or -- the fused form --
* `p2p=True` (views or tiles): the outputs live in symmetric memory
  (torch.distributed._symmetric_memory) and the render epilogue itself stores every
  value into all peers' buffers over NVLink (opts.peers of the ABI), so the exchange
  overlaps the rendering ray by ray; one device-side barrier after the launch.  The
  symmetric buffers are double-buffered (alternating calls), so the outputs of a call
  stay valid until the call after next: a fast rank's next step cannot overwrite a
  slow rank's outputs while that rank still reads them (it has to pass the next
  step's barrier first, which the slow rank reaches only after its reads, stream order).

The triplane S_t and the MLP travel together: `PackedAsset` keeps both in ONE device
buffer, so the owner's broadcast is one collective per step.

The render call is injectable (`render_fn`) so the shard/merge logic is tested on CPU
with gloo and the CPU oracle (tests/test_dist_gloo.py) and with the real kernels in two
processes on one GPU (tests/test_gpu_dist.py).
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


def tile_owner(v: int, i: int, j: int, height: int, width: int, tile: int, world: int) -> int:
    """Rank that renders pixel (v, i, j) under the interleaved-tile split."""
    th, tw = -(-height // tile), -(-width // tile)
    return ((v * th + i // tile) * tw + j // tile) % world


def peer_pointers(base_ptrs, rank: int, offset_bytes: int) -> list[int]:
    """Addresses of the same element in every other rank's symmetric buffer (bases in
    rank order), in rank order skipping `rank`."""
    return [int(b) + offset_bytes for r, b in enumerate(base_ptrs) if r != rank]


def _world(group):
    if not dist.is_initialized():
        return 1, 0
    return dist.get_world_size(group), dist.get_rank(group)


# ------------------------------------------------------------------ the asset
class PackedAsset:
    """Triplane S_t [3,R,R,C] and the shared MLP (weights W_l, fp32 biases b_l) as views
    of one device buffer, 256-byte aligned each: one broadcast moves all of them."""

    def __init__(self, triplane: torch.Tensor, mlp):
        from . import api
        parts = [triplane] + list(mlp.weights) + list(mlp.biases)
        offs, n = [], 0
        for t in parts:
            offs.append(n)
            n += (t.numel() * t.element_size() + 255) // 256 * 256
        self.flat = torch.empty(n, dtype=torch.uint8, device=triplane.device)
        views = []
        for t, o in zip(parts, offs):
            nb = t.numel() * t.element_size()
            v = self.flat[o:o + nb].view(t.dtype).view(t.shape)
            v.copy_(t)
            views.append(v)
        L = len(mlp.weights)
        self.triplane = views[0]
        self.mlp = api.DeviceMLP(views[1:1 + L], views[1 + L:], mlp.dtype, mlp.hidden_act,
                                 mlp.density_shift, mlp.rgb_widen_eps)

    @property
    def nbytes(self) -> int:
        return self.flat.numel()

    def broadcast(self, src: int = 0, group=None):
        if _world(group)[0] > 1:
            dist.broadcast(self.flat, src=src, group=group)


def _broadcast_inputs(triplane, mlp, asset, src, group, broadcast):
    if not broadcast or _world(group)[0] == 1:
        return
    if asset is not None:
        asset.broadcast(src, group)
        return
    for t in [triplane] + list(getattr(mlp, "weights", [])) + list(getattr(mlp, "biases", [])):
        if isinstance(t, torch.Tensor):  # (a host-side MLP, e.g. the oracle's, is replicated)
            dist.broadcast(t, src=src, group=group)


def _all_gather_blocks(pairs, group):
    """all_gather_into_tensor for each (full, mine) pair, coalesced into one NCCL group
    where the backend supports it; list-form fallback (e.g. gloo)."""
    if dist.get_backend(group) == "nccl":
        with dist._coalescing_manager(group=group, device=pairs[0][0].device):
            for full, mine in pairs:
                dist.all_gather_into_tensor(full, mine, group=group)
        return
    world = dist.get_world_size(group)
    for full, mine in pairs:
        parts = list(full.chunk(world))  # views into `full`: gathered in place
        dist.all_gather(parts, mine.clone(), group=group)


_SYMM = {}


def _symm_outputs(shapes, device, group):
    """Two sets of symmetric-memory output tensors (cached per shape set), alternating
    per call; returns (tensors, handles) of this call's set."""
    import torch.distributed._symmetric_memory as symm_mem
    key = (tuple(shapes), str(device), id(group))
    if key not in _SYMM:
        name = (group or dist.group.WORLD).group_name
        sets = []
        for _ in range(2):
            ts = [symm_mem.empty(*shp, dtype=torch.float32, device=device) for shp in shapes]
            sets.append((ts, [symm_mem.rendezvous(t, name) for t in ts]))
        _SYMM[key] = [sets, 0]
    sets, k = _SYMM[key]
    _SYMM[key][1] = k ^ 1
    return sets[k]


def symmetric_memory_available(device, group=None) -> bool:
    """True if symmetric-memory outputs can be set up on this group (the P2P paths)."""
    try:
        _symm_outputs([(1, 1, 8, 8)], device, group)
        return True
    except Exception:
        return False


def default_render_fn(triplane, intrinsics, c2w, height, width, mlp, alpha_bar, t, t_prev,
                      x_t, x_prev, rgb, alpha, **opts):
    from . import api
    api.dmv3d_render_ddim_step(triplane, intrinsics, c2w, height, width, mlp, alpha_bar, t,
                               t_prev, x_t, x_prev=x_prev, rgb=rgb, alpha=alpha, **opts)


# ------------------------------------------------------------------ views
def denoise_step_view_sharded(triplane, intrinsics, c2w, height, width, mlp, alpha_bar, t, t_prev,
                              x_t, ddim_views: int, group=None, src: int = 0,
                              broadcast_triplane: bool = True, render_fn=None, p2p: bool = False,
                              asset: PackedAsset | None = None, **opts):
    """One denoising step of one asset, views split across the ranks of `group`.

    Every rank passes the full `intrinsics` [V,4], `c2w` [V,3,4] and `x_t`
    [ddim_views,3,H,W]; the DDIM kwargs (eta, z, keep_mask, noise_seed, ...) are the
    one-GPU step's.  Returns (x_prev [ddim_views,3,H,W], rgb [V,3,H,W], alpha [V,H,W])
    on every rank, bitwise the one-GPU step.  `asset`: the triplane and MLP packed in
    one buffer (one broadcast); otherwise triplane and MLP tensors are broadcast one by
    one.  `p2p`: outputs assembled by the render kernel's peer stores (views valid until
    the call after next)."""
    render_fn = render_fn or default_render_fn
    world, rank = _world(group)
    if asset is not None:
        triplane, mlp = asset.triplane, asset.mlp
    _broadcast_inputs(triplane, mlp, asset, src, group, broadcast_triplane)
    V = int(c2w.shape[0])
    HW = height * width
    per = math.ceil(V / world)
    v0, v1 = view_shard(V, rank, world)
    dev = triplane.device
    nv = world * per  # padded: every rank's block has `per` views
    if p2p and world > 1:
        (xp, rgb, alpha), (hx, hr, ha) = _symm_outputs(
            [(max(ddim_views, 1), 3, height, width), (V, 3, height, width), (V, height, width)],
            dev, group)
        if v1 > v0:
            own_x = v0 < ddim_views
            peers = {"rgb": peer_pointers(hr.buffer_ptrs, rank, 0),
                     "alpha": peer_pointers(ha.buffer_ptrs, rank, 0),
                     "x_prev": peer_pointers(hx.buffer_ptrs, rank, 0) if own_x else []}
            render_fn(triplane, intrinsics, c2w, height, width, mlp, alpha_bar, t, t_prev, x_t,
                      xp[:ddim_views], rgb, alpha, ray_range=(v0 * HW, v1 * HW), peers=peers,
                      **opts)
        ha.barrier()  # every rank's peer stores have landed
        return xp[:ddim_views], rgb, alpha
    rgb = torch.empty((nv, 3, height, width), device=dev, dtype=torch.float32)
    alpha = torch.empty((nv, height, width), device=dev, dtype=torch.float32)
    xp = torch.empty((max(nv, ddim_views), 3, height, width), device=dev, dtype=torch.float32)
    if v1 > v0:
        render_fn(triplane, intrinsics, c2w, height, width, mlp, alpha_bar, t, t_prev, x_t,
                  xp[:ddim_views], rgb[:V], alpha[:V], ray_range=(v0 * HW, v1 * HW), **opts)
    if world > 1:
        blk = slice(rank * per, (rank + 1) * per)
        _all_gather_blocks([(rgb, rgb[blk]), (alpha, alpha[blk]), (xp[:nv], xp[blk])], group)
    return xp[:ddim_views], rgb[:V], alpha[:V]


# ------------------------------------------------------------------ tiles
def default_pack_fn(intrinsics, c2w, height, width, tile, rank, world, rgb, alpha, xp, prgb,
                    palpha, pxp, ddim_views):
    from . import api
    api.dmv3d_tiles_pack(intrinsics, c2w, height, width, tile, rank, world, rgb, alpha, xp, prgb,
                         palpha, pxp, ddim_views)


def default_unpack_fn(intrinsics, c2w, height, width, tile, world, prgb, palpha, pxp, rgb, alpha,
                      xp, ddim_views):
    from . import api
    api.dmv3d_tiles_unpack(intrinsics, c2w, height, width, tile, world, prgb, palpha, pxp, rgb,
                           alpha, xp, ddim_views)


def denoise_step_tile_sharded(triplane, intrinsics, c2w, height, width, mlp, alpha_bar, t, t_prev,
                              x_t, ddim_views: int, group=None, src: int = 0,
                              broadcast_triplane: bool = True, render_fn=None, tile: int = 16,
                              p2p: bool = False, asset: PackedAsset | None = None,
                              packed: bool = True, pack_fn=None, unpack_fn=None, **opts):
    """One denoising step of one asset, T x T ray tiles dealt round robin to the ranks.
    Returns the full (x_prev, rgb, alpha) on every rank.  `packed` (default): the rank's
    tiles packed (`pack_fn`, default dmv3d_tiles_pack), one all-gather, unpacked
    (`unpack_fn`, default dmv3d_tiles_unpack); `packed=False`: zeroed full-size outputs
    and one all-reduce.  `p2p`: outputs in symmetric
    memory, every rank's render epilogue stores its pixels into all peers' buffers at the
    same offsets (no collective on the data path; one device-side barrier; views valid
    until the call after next)."""
    render_fn = render_fn or default_render_fn
    world, rank = _world(group)
    if asset is not None:
        triplane, mlp = asset.triplane, asset.mlp
    _broadcast_inputs(triplane, mlp, asset, src, group, broadcast_triplane)
    V = int(c2w.shape[0])
    dev = triplane.device
    if p2p and world > 1:
        (xp, rgb, alpha), (hx, hr, ha) = _symm_outputs(
            [(max(ddim_views, 1), 3, height, width), (V, 3, height, width), (V, height, width)],
            dev, group)
        peers = {"rgb": peer_pointers(hr.buffer_ptrs, rank, 0),
                 "alpha": peer_pointers(ha.buffer_ptrs, rank, 0),
                 "x_prev": peer_pointers(hx.buffer_ptrs, rank, 0)}
        render_fn(triplane, intrinsics, c2w, height, width, mlp, alpha_bar, t, t_prev, x_t,
                  xp[:ddim_views], rgb, alpha, tiles=(tile, rank, world), peers=peers, **opts)
        ha.barrier()
        return xp[:ddim_views], rgb, alpha
    HW = height * width
    if packed:
        # the rank renders its tiles into image-layout scratch, dmv3d_tiles_pack copies them
        # into its blocks (rgb [k][3][T][T], alpha [k][T][T], x_prev [k][3][T][T]), one
        # coalesced all-gather stacks the ranks' blocks, dmv3d_tiles_unpack scatters them
        pack_fn = pack_fn or default_pack_fn
        unpack_fn = unpack_fn or default_unpack_fn
        xp = torch.empty((ddim_views, 3, height, width), device=dev, dtype=torch.float32)
        rgb = torch.empty((V, 3, height, width), device=dev, dtype=torch.float32)
        alpha = torch.empty((V, height, width), device=dev, dtype=torch.float32)
        render_fn(triplane, intrinsics, c2w, height, width, mlp, alpha_bar, t, t_prev, x_t, xp, rgb,
                  alpha, tiles=(tile, rank, world), **opts)
        if world == 1:
            return xp, rgb, alpha
        nmax = -(-(V * -(-height // tile) * -(-width // tile)) // world)
        g_rgb = torch.empty((world * nmax, 3, tile, tile), device=dev, dtype=torch.float32)
        g_a = torch.empty((world * nmax, tile, tile), device=dev, dtype=torch.float32)
        g_x = torch.empty((world * nmax, 3, tile, tile), device=dev, dtype=torch.float32)
        blk = slice(rank * nmax, (rank + 1) * nmax)
        pack_fn(intrinsics, c2w, height, width, tile, rank, world, rgb, alpha, xp, g_rgb[blk], g_a[blk],
                g_x[blk], ddim_views)
        _all_gather_blocks([(g_rgb, g_rgb[blk]), (g_a, g_a[blk]), (g_x, g_x[blk])], group)
        unpack_fn(intrinsics, c2w, height, width, tile, world, g_rgb, g_a, g_x, rgb, alpha, xp,
                  ddim_views)
        return xp, rgb, alpha
    n_x, n_rgb = ddim_views * 3 * HW, V * 3 * HW
    flat = torch.zeros(n_x + n_rgb + V * HW, device=dev, dtype=torch.float32)  # one collective
    xp = flat[:n_x].view(ddim_views, 3, height, width)
    rgb = flat[n_x:n_x + n_rgb].view(V, 3, height, width)
    alpha = flat[n_x + n_rgb:].view(V, height, width)
    render_fn(triplane, intrinsics, c2w, height, width, mlp, alpha_bar, t, t_prev, x_t, xp, rgb,
              alpha, tiles=(tile, rank, world), **opts)
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


def sum_over_ranks(values, device, group=None):
    """Per-rank counters (e.g. the kernel's hit / evaluated-sample counters) summed."""
    t = torch.as_tensor(values, dtype=torch.float64, device=device).clone()
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t.cpu().numpy()
