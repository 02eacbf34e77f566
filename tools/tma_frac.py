"""Fraction of cfg3 blend windows staged by TMA boxes (counters[6] / blend windows)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_18052_b200 import api, workloads as wl  # noqa: E402

w = wl.make_workload("cfg3")
dev = torch.device("cuda")
tp = torch.from_numpy(w.triplane).to(dev).to(torch.bfloat16)
intr = torch.from_numpy(w.cameras.intrinsics).to(dev)
c2w = torch.from_numpy(w.cameras.c2w).to(dev)
mlp = api.DeviceMLP.from_host(w.mlp, "bf16", dev)
cnt = torch.zeros(8, dtype=torch.int64, device=dev)
api.dmv3d_render_views(tp, intr, c2w, 256, 256, mlp, samples_per_ray=128, term_eps=1e-4,
                       engine="tcgen05", counters=cnt)
c = cnt.cpu().numpy()
print("blend windows", c[4] // 128, "TMA-staged", c[6], "fraction", c[6] / max(c[4] / 128, 1))
