"""Probe: central differences of L = <g, rgb> + <gA, alpha> (fp32 SIMT forward) along a
random direction of one weight matrix, at several step sizes, against the SIMT and TC
backward's directional derivatives (cfg2 size)."""
import sys
import torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from paper_2605_18052_b200 import api, workloads as wl  # noqa: E402
from helpers import dev_workload  # noqa: E402
w = wl.make_workload("cfg2_bf16")
V, H, W, N = w.cameras.num_views, w.cameras.height, w.cameras.width, w.samples_per_ray
t, intr, c2w, mlp = dev_workload(w)
gen = torch.Generator(device="cuda").manual_seed(5)
g = torch.randn((V, 3, H, W), device="cuda", generator=gen)
gA = torch.randn((V, H, W), device="cuda", generator=gen)
tc = api.dmv3d_render_backward(t, intr, c2w, H, W, mlp, g, gA, samples_per_ray=N, engine="tcgen05")
si = api.dmv3d_render_backward(t, intr, c2w, H, W, mlp, g, gA, samples_per_ray=N, engine="simt")
w32 = [x.float() for x in mlp.weights]
tp32 = t.float()


def loss(ws_):
    m = api.DeviceMLP(ws_, mlp.biases, "f32")
    rgb, alpha = api.dmv3d_render_views(tp32, intr, c2w, H, W, m, samples_per_ray=N, engine="simt")
    return float((g.double() * rgb.double()).sum() + (gA.double() * alpha.double()).sum())


for l in range(4):
    d = torch.randn(w32[l].shape, device="cuda", generator=gen)
    d = d / d.abs().max()
    out = [f"W{l}: tc {float((tc[1][l].double() * d.double()).sum()):.5g}",
           f"simt {float((si[1][l].double() * d.double()).sum()):.5g}"]
    for eps in (1e-2, 3e-3, 1e-3, 3e-4, 1e-4):
        ws_p, ws_m = list(w32), list(w32)
        ws_p[l] = w32[l] + eps * d
        ws_m[l] = w32[l] - eps * d
        out.append(f"fd({eps:g}) {(loss(ws_p) - loss(ws_m)) / (2 * eps):.5g}")
    print("  ".join(out))
