"""Multi-process (world_size 2, gloo, CPU) tests of the sharding/merge logic in
paper_2605_18052_b200.dist, with the CPU oracle standing in for the renderer:
the gathered views equal one process rendering everything (bitwise) -- also with
the DDIM keep-mask and eta > 0, whose view indices must stay global on every rank --,
the triplane broadcast reaches every rank, and asset shards cover the batch."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_18052_b200 import dist as pdist
from paper_2605_18052_b200 import schedule
from paper_2605_18052_b200 import workloads as wl


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _workload():
    tp = wl.blob_triplane(8, 8, seed=3, kappa=4.0)
    m = wl.blob_mlp(8, 16, 3, seed=4)
    cams = wl.concat_cameras(wl.input_cameras(6, 5, 3), wl.novel_cameras(6, 5, 2, seed=5))
    return tp, m, cams


def _oracle_render_fn(triplane, intrinsics, c2w, H, W, mlp, alpha_bar, t, t_prev, x_t, x_prev, rgb,
                      alpha, samples_per_ray=16, ray_range=None, eta=0.0, z=None, keep_mask=None):
    """The oracle as the fused step over the FULL camera set, writing only the views of
    `ray_range` (whole views), with the one-GPU step's DDIM arguments."""
    import oracle
    cams = wl.Cameras(intrinsics.numpy(), c2w.numpy(), H, W)
    orgb, oalpha = oracle.render_views(triplane.numpy(), cams, mlp, samples_per_ray, threads=1)
    V = orgb.shape[0]
    v0, v1 = (0, V) if ray_range is None else (ray_range[0] // (H * W), ray_range[1] // (H * W))
    rgb[v0:v1] = torch.from_numpy(orgb[v0:v1].astype(np.float32))
    alpha[v0:v1] = torch.from_numpy(oalpha[v0:v1].astype(np.float32))
    if x_t is not None:
        dv = x_t.shape[0]
        xp = oracle.ddim_step(alpha_bar, t, t_prev, x_t.numpy(), orgb[:dv], eta=eta,
                              z=None if z is None else z.numpy(), keep_mask=keep_mask)
        x_prev[v0:min(v1, dv)] = torch.from_numpy(xp[v0:min(v1, dv)].astype(np.float32))


def _oracle_tile_render_fn(triplane, intrinsics, c2w, H, W, mlp, alpha_bar, t, t_prev, x_t, x_prev,
                           rgb, alpha, tiles, samples_per_ray=16):
    """The oracle as a tile-sharded renderer: writes only the pixels of this rank's tiles
    (ownership from the tile formula written out here, independently of dist.py)."""
    T, rank, world = tiles
    full_rgb, full_a = torch.zeros_like(rgb), torch.zeros_like(alpha)
    full_x = torch.zeros_like(x_prev) if x_prev is not None else None
    _oracle_render_fn(triplane, intrinsics, c2w, H, W, mlp, alpha_bar, t, t_prev, x_t, full_x,
                      full_rgb, full_a, samples_per_ray)
    V = rgb.shape[0]
    th, tw = -(-H // T), -(-W // T)
    for v in range(V):
        for i in range(H):
            for j in range(W):
                if ((v * th + i // T) * tw + j // T) % world == rank:
                    rgb[v, :, i, j] = full_rgb[v, :, i, j]
                    alpha[v, i, j] = full_a[v, i, j]
                    if x_prev is not None and v < x_prev.shape[0]:
                        x_prev[v, :, i, j] = full_x[v, :, i, j]


def _tile_blocks(V, H, W, T, world):
    """(rank, block k, view, tile row, tile col) of every tile, from the tile formula
    tau = (v th + i / T) tw + j / T written out here: rank tau mod P, block tau div P."""
    th, tw = -(-H // T), -(-W // T)
    for tau in range(V * th * tw):
        v, rem = divmod(tau, th * tw)
        yield tau % world, tau // world, v, rem // tw, rem % tw


def _loop_pack_fn(intrinsics, c2w, H, W, T, rank, world, rgb, alpha, xp, prgb, palpha, pxp, ddim_views):
    for r, k, v, ti, tj in _tile_blocks(c2w.shape[0], H, W, T, world):
        if r != rank:
            continue
        for pi in range(T):
            for pj in range(T):
                i, j = ti * T + pi, tj * T + pj
                if i < H and j < W:
                    prgb[k, :, pi, pj] = rgb[v, :, i, j]
                    palpha[k, pi, pj] = alpha[v, i, j]
                    if v < ddim_views:
                        pxp[k, :, pi, pj] = xp[v, :, i, j]


def _loop_unpack_fn(intrinsics, c2w, H, W, T, world, prgb, palpha, pxp, rgb, alpha, xp, ddim_views):
    nmax = prgb.shape[0] // world
    for r, k, v, ti, tj in _tile_blocks(c2w.shape[0], H, W, T, world):
        b = r * nmax + k
        for pi in range(T):
            for pj in range(T):
                i, j = ti * T + pi, tj * T + pj
                if i < H and j < W:
                    rgb[v, :, i, j] = prgb[b, :, pi, pj]
                    alpha[v, i, j] = palpha[b, pi, pj]
                    if v < ddim_views:
                        xp[v, :, i, j] = pxp[b, :, pi, pj]


def _tile_worker(rank, world, port, out_dir, packed=True):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        tp, m, cams = _workload()
        triplane = torch.from_numpy(tp) if rank == 0 else torch.zeros_like(torch.from_numpy(tp))
        x_t = torch.from_numpy(wl.gaussian((3, 3, 6, 5), 4))
        xp, rgb, alpha = pdist.denoise_step_tile_sharded(
            triplane, torch.from_numpy(cams.intrinsics), torch.from_numpy(cams.c2w), 6, 5, m,
            schedule.cosine_alpha_bar(), 980, 960, x_t, ddim_views=3,
            render_fn=_oracle_tile_render_fn, tile=4, samples_per_ray=16, packed=packed,
            pack_fn=_loop_pack_fn, unpack_fn=_loop_unpack_fn)
        np.savez(os.path.join(out_dir, f"t{rank}.npz"), xp=xp.numpy(), rgb=rgb.numpy(),
                 alpha=alpha.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("packed", [True, False], ids=["all-gather", "all-reduce"])
def test_tile_sharded_step_matches_single_process(tmp_path, packed):
    world = 2
    mp.spawn(_tile_worker, args=(world, _free_port(), str(tmp_path), packed), nprocs=world, join=True)
    import oracle
    tp, m, cams = _workload()
    orgb, oalpha = oracle.render_views(tp, cams, m, 16, threads=1)
    oxp = oracle.ddim_step(schedule.cosine_alpha_bar(), 980, 960, wl.gaussian((3, 3, 6, 5), 4), orgb[:3])
    for r in range(world):
        d = np.load(tmp_path / f"t{r}.npz")
        assert np.array_equal(d["rgb"], orgb.astype(np.float32))
        assert np.array_equal(d["alpha"], oalpha.astype(np.float32))
        assert np.array_equal(d["xp"], oxp.astype(np.float32))


@pytest.mark.parametrize("H,W,T,P", [(6, 5, 4, 2), (16, 16, 4, 3), (33, 20, 8, 4)])
def test_tile_owner_partition(H, W, T, P):
    """Every pixel has one owner; owners cycle over consecutive tiles."""
    owners = np.array([[[pdist.tile_owner(v, i, j, H, W, T, P) for j in range(W)] for i in range(H)]
                       for v in range(3)])
    assert owners.min() >= 0 and owners.max() < P
    assert owners[0, 0, 0] == 0 and (W > T) == (owners[0, 0, min(T, W - 1)] == 1 % P)


DDIM_KW = {"plain": {}, "keep_eta": {"eta": 1.0, "keep_mask": [0, 0, 1]}}


def _worker(rank, world, port, out_dir, case="plain"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        tp, m, cams = _workload()
        triplane = torch.from_numpy(tp) if rank == 0 else torch.zeros_like(torch.from_numpy(tp))
        ab = schedule.cosine_alpha_bar()
        x_t = torch.from_numpy(wl.gaussian((3, 3, 6, 5), 4))
        kw = dict(DDIM_KW[case])
        if kw.get("eta"):
            kw["z"] = torch.from_numpy(wl.gaussian((3, 3, 6, 5), 9))
        xp, rgb, alpha = pdist.denoise_step_view_sharded(
            triplane, torch.from_numpy(cams.intrinsics), torch.from_numpy(cams.c2w), 6, 5, m, ab,
            980, 960, x_t, ddim_views=3, render_fn=_oracle_render_fn, samples_per_ray=16, **kw)
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), xp=xp.numpy(), rgb=rgb.numpy(),
                 alpha=alpha.numpy(), tp=triplane.numpy(),
                 t=np.array([pdist.max_over_ranks(float(rank + 1), "cpu")]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", ["plain", "keep_eta"])
def test_view_sharded_step_matches_single_process(tmp_path, case):
    """Rank 1 owns views 3-4: a novel view and the last DDIM view (which is the kept
    one in "keep_eta"), so keep_mask / z / x_t must be read at global view indices."""
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path), case), nprocs=world, join=True)
    import oracle
    tp, m, cams = _workload()
    orgb, oalpha = oracle.render_views(tp, cams, m, 16, threads=1)
    x_t = wl.gaussian((3, 3, 6, 5), 4)
    kw = dict(DDIM_KW[case])
    if kw.get("eta"):
        kw["z"] = wl.gaussian((3, 3, 6, 5), 9)
    oxp = oracle.ddim_step(schedule.cosine_alpha_bar(), 980, 960, x_t, orgb[:3], **kw)
    for r in range(world):
        d = np.load(tmp_path / f"r{r}.npz")
        assert np.array_equal(d["tp"], tp)  # broadcast from the owner rank
        assert np.array_equal(d["rgb"], orgb.astype(np.float32))
        assert np.array_equal(d["alpha"], oalpha.astype(np.float32))
        assert np.array_equal(d["xp"], oxp.astype(np.float32))
        assert d["t"][0] == world  # max over ranks


@pytest.mark.parametrize("V,P", [(8, 1), (8, 2), (8, 8), (5, 2), (3, 4), (7, 3)])
def test_view_shard_partition(V, P):
    blocks = [pdist.view_shard(V, r, P) for r in range(P)]
    covered = [v for b in blocks for v in range(*b)]
    assert covered == list(range(V))
    per = -(-V // P)
    assert all(b[1] - b[0] <= per for b in blocks)


def test_asset_shard_partition():
    owned = sorted(a for r in range(3) for a in pdist.asset_shard(8, r, 3))
    assert owned == list(range(8))


def test_peer_pointers_skip_own_rank():
    """P2P view sharding: each peer gets the same element offset in its own buffer."""
    from paper_2605_18052_b200.dist import peer_pointers
    bases = [1000, 5000, 9000, 13000]
    assert peer_pointers(bases, 1, 64) == [1064, 9064, 13064]
    assert peer_pointers(bases, 0, 0) == [5000, 9000, 13000]
    assert peer_pointers([7], 0, 4) == []
