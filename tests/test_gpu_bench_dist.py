"""bench.py's N > 1 path end to end: torchrun with two ranks sharing cuda:0 (gloo, since
NCCL refuses two ranks on one device).  The line must be the strong-scaling single-asset
step (view split: packed triplane + MLP broadcast and all-gather inside the timed region)
with honest units: one asset's rays per step, counters summed over the ranks, and the
weak-scaling asset split as an extra key."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("mode", ["views", "tiles"])
def test_torchrun_two_ranks_prints_one_strong_scaling_line(mode):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py",
           "--gpus", "2", "--share-gpu", "--steps", "3", "--warmup", "3", "--no-cpu-baseline",
           "--sustained-s", "0", "--config", "cfg2", "--mode", mode]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["config"]["assets"] == 1 and d["config"]["rays_per_step"] == 4 * 128 * 128
    assert d["value"] > 0 and d["e2e"]["value"] > 0
    # one asset's rays: the evaluated fraction is a fraction (counters summed over ranks)
    assert 0.3 < d["evaluated_fraction_of_nominal"] < 1.0
    assert 0.5 < d["hit_fraction"] <= 1.0
    assert d["weak_assets"]["assets"] == 2 and d["weak_assets"]["value"] > 0
    assert "broadcast" in d["config"]["parallelism"]
