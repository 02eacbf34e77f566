"""The multi-GPU step functions with the REAL CUDA render, in two processes.

Only one GPU is available to the build, so both ranks run on cuda:0 and talk over
gloo (NCCL refuses two ranks on one device).  Each rank gets the asset (triplane +
MLP, one PackedAsset buffer) by broadcast from rank 0, renders its share -- interleaved
16x16... here 8x8 ray tiles, or a block of views -- through libdmv3d, and the merge
(all-reduce / all-gather) assembles the step.  The result must be BITWISE the
one-process step (SURVEY §8c pin P12), including eta > 0 with z and a keep-mask whose
kept view belongs to rank 1 (global view indices on every rank)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_18052_b200 import api, schedule
from paper_2605_18052_b200 import dist as pdist
from paper_2605_18052_b200 import workloads as wl

pytestmark = pytest.mark.gpu
H = W = 32
DV = 4
KW = dict(samples_per_ray=48, term_eps=1e-4, eta=1.0, keep_mask=[0, 0, 0, 1])


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _inputs(dev):
    tp = wl.round_to_bf16(wl.blob_triplane(32, 32, seed=5))
    m = wl.bf16_mlp(wl.blob_mlp(32, 64, 4, seed=6))
    cams = wl.concat_cameras(wl.input_cameras(H, W, DV), wl.novel_cameras(H, W, 2, seed=7))
    return (torch.from_numpy(tp).to(dev).to(torch.bfloat16).contiguous(),
            api.DeviceMLP.from_host(m, "bf16", dev), torch.from_numpy(cams.intrinsics).to(dev),
            torch.from_numpy(cams.c2w).to(dev), torch.from_numpy(wl.gaussian((DV, 3, H, W), 8)).to(dev),
            torch.from_numpy(wl.gaussian((DV, 3, H, W), 9)).to(dev))


def _worker(rank, world, port, out_dir, engine):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        tp, mlp, intr, c2w, x_t, z = _inputs(dev)
        asset = pdist.PackedAsset(tp if rank == 0 else torch.zeros_like(tp),
                                  mlp if rank == 0 else api.DeviceMLP(
                                      [torch.zeros_like(w) for w in mlp.weights],
                                      [torch.zeros_like(b) for b in mlp.biases], "bf16"))
        ab = schedule.cosine_alpha_bar()
        out = {}
        for name, fn, extra in (("tiles", pdist.denoise_step_tile_sharded, {"tile": 8}),
                                ("views", pdist.denoise_step_view_sharded, {})):
            xp, rgb, alpha = fn(None, intr, c2w, H, W, None, ab, 500, 480, x_t, DV, asset=asset,
                                z=z, engine=engine, **extra, **KW)
            torch.cuda.synchronize()
            out[name + "_xp"], out[name + "_rgb"] = xp.cpu().numpy(), rgb.cpu().numpy()
            out[name + "_alpha"] = alpha.cpu().numpy()
        out["tp"] = asset.triplane.float().cpu().numpy()
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), **out)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("engine", ["tcgen05", "simt"])
def test_two_process_steps_are_the_one_gpu_step(tmp_path, engine):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path), engine), nprocs=world, join=True)
    dev = torch.device("cuda", 0)
    tp, mlp, intr, c2w, x_t, z = _inputs(dev)
    xp, rgb, alpha = api.dmv3d_render_ddim_step(tp, intr, c2w, H, W, mlp, schedule.cosine_alpha_bar(),
                                                500, 480, x_t, z=z, engine=engine, **KW)
    ref = {"xp": xp.cpu().numpy(), "rgb": rgb.cpu().numpy(), "alpha": alpha.cpu().numpy()}
    for r in range(world):
        d = np.load(tmp_path / f"r{r}.npz")
        assert np.array_equal(d["tp"], tp.float().cpu().numpy())  # the broadcast
        for split in ("tiles", "views"):
            for k in ("xp", "rgb", "alpha"):
                assert np.array_equal(d[f"{split}_{k}"], ref[k]), (r, split, k)
