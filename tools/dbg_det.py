import sys; sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/tests')
import torch, numpy as np
from paper_2605_18052_b200 import api, workloads as wl
from helpers import dev_workload
from test_gpu_tc import _wl
w = _wl(C=32, L=4, H=24, W=28, N=40)
tp, intr, c2w, mlp = dev_workload(w)
H, W = 24, 28
kw = dict(samples_per_ray=40, term_eps=1e-4, engine="tcgen05")
outs=[api.dmv3d_render_views(tp, intr, c2w, H, W, mlp, **kw) for _ in range(4)]
for o in outs[1:]:
    d=(o[0]-outs[0][0]).abs(); print('rgb diff max', d.max().item(), 'n', (d>0).sum().item(), 'alpha', (o[1]-outs[0][1]).abs().max().item())
    idx=(d>0).nonzero()[:5]; print(idx.tolist())
c = torch.full_like(outs[0][0], -7.0); cc = torch.full_like(outs[0][1], -7.0)
cuts = [0, 500, H * W, H * W + 333, w.num_rays]
for lo, hi in zip(cuts[:-1], cuts[1:]):
    api.dmv3d_render_views(tp, intr, c2w, H, W, mlp, rgb=c, alpha=cc, ray_range=(lo, hi), **kw)
d=(c-outs[0][0]).abs(); print('shard diff', d.max().item(), (d>0).sum().item(), (c==-7).sum().item())
idx=(d>0).nonzero()[:10]; print(idx.tolist())
# simt vs itself
a=api.dmv3d_render_views(tp, intr, c2w, H, W, mlp, samples_per_ray=40, term_eps=1e-4, engine="simt")
b=api.dmv3d_render_views(tp, intr, c2w, H, W, mlp, samples_per_ray=40, term_eps=1e-4, engine="simt")
print('simt det', (a[0]-b[0]).abs().max().item())
