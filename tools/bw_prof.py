"""Small renderer-backward workload for ncu (2 views 128^2, cfg2 triplane/MLP, N = 128).
    python tools/bw_prof.py [simt|tcgen05]"""
import sys

import torch

sys.path.insert(0, '.')
from paper_2605_18052_b200 import api  # noqa: E402
from paper_2605_18052_b200 import workloads as wl  # noqa: E402

engine = sys.argv[1] if len(sys.argv) > 1 else "simt"
w = wl.make_workload("cfg2")
dev = torch.device("cuda", 0)
tp = torch.from_numpy(w.triplane).to(dev).to(torch.bfloat16).contiguous()
m = api.DeviceMLP.from_host(wl.bf16_mlp(w.mlp), "bf16", dev)
cams = wl.input_cameras(128, 128, 2)
intr = torch.from_numpy(cams.intrinsics).to(dev)
c2w = torch.from_numpy(cams.c2w).to(dev)
g = torch.randn((2, 3, 128, 128), device=dev)
gA = torch.randn((2, 128, 128), device=dev)
for _ in range(2):
    api.dmv3d_render_backward(tp, intr, c2w, 128, 128, m, g, gA, samples_per_ray=128, engine=engine)
torch.cuda.synchronize()
