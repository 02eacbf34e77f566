"""GPU parity of the SURVEY §8(f) rows against the oracle (-m gpu):
f2 Plucker ray map (bit-exact), f3 density grid (fp32 bar)."""
import numpy as np
import pytest
import torch

import oracle
from paper_2605_18052_b200 import api, schedule
from paper_2605_18052_b200 import workloads as wl

from helpers import dev_cams, dev_workload

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _cams():
    return wl.concat_cameras(wl.concat_cameras(wl.input_cameras(11, 13, 4),
                                               wl.novel_cameras(11, 13, 3, seed=5)),
                             wl.axis_camera(11, 13))


def test_plucker_standalone_bit_exact():
    cams = _cams()
    intr, c2w = dev_cams(cams)
    g = api.dmv3d_plucker_rays(intr, c2w, 11, 13).cpu().numpy()  # [V,6,H,W]
    ids = np.arange(cams.num_views * 143)
    want = oracle.plucker(cams, ids)  # [n,6]
    got = g.transpose(0, 2, 3, 1).reshape(-1, 6)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


@pytest.mark.parametrize("H,W,rng", [(16, 12, None), (16, 12, (4, 1532)), (16, 12, (3, 1001)),
                                     (9, 7, (10, 400))],
                         ids=["vec", "vec-range", "scalar-range", "scalar-ragged"])
def test_plucker_standalone_paths_bit_exact(H, W, rng):
    """The float4 path (H W % 4 == 0, 4-aligned ray range) and the scalar path, with ray
    ranges that start and end inside a view: bit-exact against the oracle, pixels outside
    the range untouched."""
    cams = wl.concat_cameras(wl.input_cameras(H, W, 4), wl.novel_cameras(H, W, 4, seed=9))
    intr, c2w = dev_cams(cams)
    out = torch.full((8, 6, H, W), -7.0, device="cuda")
    api.dmv3d_plucker_rays(intr, c2w, H, W, out=out, ray_range=rng)
    g = out.cpu().numpy().transpose(0, 2, 3, 1).reshape(-1, 6)
    n = 8 * H * W
    lo, hi = rng if rng else (0, n)
    want = oracle.plucker(cams, np.arange(lo, hi))
    assert np.array_equal(g[lo:hi].view(np.uint32), want.view(np.uint32))
    assert (g[:lo] == -7.0).all() and (g[hi:] == -7.0).all()


@pytest.mark.parametrize("V,H,W,rng", [(10, 512, 512, None), (10, 510, 251, None),
                                       (10, 512, 512, (1024, 2600000))],
                         ids=["float4", "float2", "float4-range"])
def test_plucker_standalone_wide_stores_bit_exact(V, H, W, rng):
    """Launches big enough for 4 / 2 rays per thread (float4 / float2 planar stores):
    a seeded subset of 20k rays (plus both ends of the range) bit-exact against the
    oracle, every value in the range written, the rest untouched."""
    cams = wl.concat_cameras(wl.input_cameras(H, W, 4), wl.novel_cameras(H, W, V - 4, seed=9))
    intr, c2w = dev_cams(cams)
    out = torch.full((V, 6, H, W), float("nan"), device="cuda")
    api.dmv3d_plucker_rays(intr, c2w, H, W, out=out, ray_range=rng)
    g = out.permute(0, 2, 3, 1).reshape(-1, 6).cpu().numpy()
    n = V * H * W
    lo, hi = rng if rng else (0, n)
    ids = np.unique(np.concatenate([np.random.default_rng(5).integers(lo, hi, 20000), [lo, hi - 1]]))
    want = oracle.plucker(cams, ids)
    assert np.array_equal(g[ids].view(np.uint32), want.view(np.uint32))
    assert np.isfinite(g[lo:hi]).all()
    assert np.isnan(g[:lo]).all() and np.isnan(g[hi:]).all()


@pytest.mark.parametrize("engine,dtype", [("simt", "f32"), ("tcgen05", "bf16")])
def test_plucker_emitted_by_the_renderer(engine, dtype):
    tp = wl.blob_triplane(16, 32, seed=2)
    m = wl.blob_mlp(32, 64, 4, seed=3)
    if dtype == "bf16":
        tp, m = wl.round_to_bf16(tp), wl.bf16_mlp(m)
    cams = _cams()
    w = wl.Workload("pl", tp, cams, m, 24, dtype)
    t, intr, c2w, mlp = dev_workload(w)
    pl = torch.full((cams.num_views, 6, 11, 13), -5.0, device="cuda")
    api.dmv3d_render_views(t, intr, c2w, 11, 13, mlp, samples_per_ray=24, engine=engine, plucker=pl)
    ref = api.dmv3d_plucker_rays(intr, c2w, 11, 13)
    assert torch.equal(pl, ref)


@pytest.mark.parametrize("G,dtype,engine", [(9, "f32", "simt"), (20, "f32", "simt"),
                                            (33, "bf16", "simt"), (33, "bf16", "tcgen05"),
                                            (70, "bf16", "tcgen05")])
def test_density_grid_matches_oracle(G, dtype, engine):
    tp = wl.blob_triplane(12, 32, seed=4)
    m = wl.blob_mlp(32, 64, 4, seed=5)
    if dtype == "bf16":
        tp, m = wl.round_to_bf16(tp), wl.bf16_mlp(m)
    dt = torch.bfloat16 if dtype == "bf16" else torch.float32
    sigma, rgb = api.dmv3d_density_grid(torch.from_numpy(tp).cuda().to(dt),
                                        api.DeviceMLP.from_host(m, dtype), G, engine=engine)
    osig, orgb = oracle.density_grid(tp, m, G)
    s = sigma.cpu().numpy()
    # fp32 engine: 1e-5; tensor-core engine (fp16 MMAs): the 2e-2 bar on the decoded values
    tol = 1e-5 if engine == "simt" else 2e-2
    assert np.all(s > 0) and np.all(np.isfinite(s))  # softplus > 0: every point written
    assert np.max(np.abs(s - osig) / np.maximum(1.0, osig)) < tol
    assert np.max(np.abs(rgb.cpu().numpy() - orgb)) < tol
    # the blob is a ball: the level set sigma = 1 encloses the centre, not the corners
    c = G // 2
    assert s[c, c, c] > 1.0 and s[0, 0, 0] < 1.0


def test_in_kernel_noise_ddim_matches_oracle():
    """Row f4: eta = 1 with the noise drawn in the kernel (standalone and fused, both
    engines) equals the oracle's DDIM step with the oracle's copy of the generator."""
    from paper_2605_18052_b200 import schedule
    ab = schedule.cosine_alpha_bar()
    V, H, W = 2, 12, 12
    x_t = wl.gaussian((V, 3, H, W), 4)
    rgb = np.random.default_rng(3).uniform(size=(V, 3, H, W)).astype(np.float32)
    z = oracle.noise(77, V * 3 * H * W).reshape(V, 3, H, W)
    want = oracle.ddim_step(oracle.cosine_alpha_bar(), 500, 480, x_t, rgb, z, eta=1.0)
    g = api.dmv3d_ddim_step(ab, 500, 480, torch.from_numpy(x_t).cuda(), torch.from_numpy(rgb).cuda(),
                            None, 1.0, noise_seed=77).cpu().numpy()
    assert np.max(np.abs(g - want)) < 1e-5
    for engine, dtype in (("simt", "f32"), ("tcgen05", "bf16")):
        tp = wl.blob_triplane(12, 32, seed=2)
        m = wl.blob_mlp(32, 64, 4, seed=3)
        if dtype == "bf16":
            tp, m = wl.round_to_bf16(tp), wl.bf16_mlp(m)
        cams = wl.input_cameras(H, W, V)
        w = wl.Workload("nz", tp, cams, m, 32, dtype)
        t, intr, c2w, mlp = dev_workload(w)
        xp, r, a = api.dmv3d_render_ddim_step(t, intr, c2w, H, W, mlp, ab, 500, 480,
                                              torch.from_numpy(x_t).cuda(), None, 1.0,
                                              samples_per_ray=32, engine=engine, noise_seed=77)
        orgb, _ = oracle.render_views(tp, cams, m, 32)
        want = oracle.ddim_step(oracle.cosine_alpha_bar(), 500, 480, x_t, orgb, z, eta=1.0)
        tol = 1e-4 if engine == "simt" else 5e-2
        assert np.max(np.abs(xp.cpu().numpy() - want)) < tol, engine


def _close(g, o, rel=1e-4):
    g, o = np.asarray(g, np.float64), np.asarray(o, np.float64)
    return np.max(np.abs(g - o)) <= rel * max(np.max(np.abs(o)), 1e-30) + 1e-7


@pytest.mark.parametrize("C,H,L,dtype,agg", [(32, 64, 4, "f32", "mean"), (80, 64, 4, "bf16", "mean"),
                                              (16, 32, 3, "f32", "sum"), (8, 16, 2, "f32", "mean")])
def test_render_backward_matches_oracle(C, H, L, dtype, agg):
    """Row f1: triplane and MLP gradients of <g, rgb> + <gA, alpha> vs the oracle's
    (finite-difference-pinned) analytic backward; fp32 with atomics: 1e-4 relative."""
    tp = wl.blob_triplane(12, C, seed=7, kappa=4.0)
    m = wl.blob_mlp(C, H, L, seed=8)
    if dtype == "bf16":
        tp, m = wl.round_to_bf16(tp), wl.bf16_mlp(m)
    cams = wl.concat_cameras(wl.input_cameras(10, 9, 2), wl.novel_cameras(10, 9, 1, seed=9))
    w = wl.Workload("bw", tp, cams, m, 40, dtype)
    t, intr, c2w, mlp = dev_workload(w)
    rng = np.random.default_rng(C)
    g = rng.normal(size=(3, 3, 10, 9)).astype(np.float32)
    gA = rng.normal(size=(3, 10, 9)).astype(np.float32)
    dF, dW, db = api.dmv3d_render_backward(t, intr, c2w, 10, 9, mlp, torch.from_numpy(g).cuda(),
                                           torch.from_numpy(gA).cuda(), samples_per_ray=40,
                                           agg=agg, bg=(0.3, 0.5, 0.7))
    oagg = oracle.AGG_MEAN if agg == "mean" else oracle.AGG_SUM
    oF, oW, ob = oracle.render_backward(tp, cams, m, 40, g, gA, agg=oagg, bg=(0.3, 0.5, 0.7))
    assert np.max(np.abs(oF)) > 0
    assert _close(dF.cpu().numpy(), oF)
    for l in range(L):
        assert _close(dW[l].cpu().numpy(), oW[l]), l
        assert _close(db[l].cpu().numpy(), ob[l]), l


@pytest.mark.parametrize("engine,dtype", [("simt", "f32"), ("tcgen05", "bf16")])
def test_peer_stores_write_every_copy(engine, dtype):
    """opts.peers (view-sharded multi-GPU step): every rgb / alpha / x_prev value the
    render epilogue writes is also stored at the same offset of each peer buffer.  On one
    GPU the peers are local buffers; the values must equal the local output bitwise."""
    from paper_2605_18052_b200 import schedule
    tp = wl.blob_triplane(12, 32, seed=2)
    m = wl.blob_mlp(32, 64, 4, seed=3)
    if dtype == "bf16":
        tp, m = wl.round_to_bf16(tp), wl.bf16_mlp(m)
    cams = wl.concat_cameras(wl.input_cameras(12, 10, 2), wl.novel_cameras(12, 10, 2, seed=4))
    w = wl.Workload("peer", tp, cams, m, 24, dtype)
    t, intr, c2w, mlp = dev_workload(w)
    V, H, W = 4, 12, 10
    x_t = torch.from_numpy(wl.gaussian((2, 3, H, W), 4)).cuda()
    peer_rgb = [torch.full((V, 3, H, W), -1.0, device="cuda") for _ in range(3)]
    peer_a = [torch.full((V, H, W), -1.0, device="cuda") for _ in range(3)]
    peer_x = [torch.full((2, 3, H, W), -1.0, device="cuda") for _ in range(3)]
    peers = {"rgb": [p.data_ptr() for p in peer_rgb], "alpha": [p.data_ptr() for p in peer_a],
             "x_prev": [p.data_ptr() for p in peer_x[:2]] + [0]}  # third peer skips x_prev
    xp, rgb, alpha = api.dmv3d_render_ddim_step(t, intr, c2w, H, W, mlp, schedule.cosine_alpha_bar(),
                                                980, 960, x_t, samples_per_ray=24, engine=engine,
                                                peers=peers)
    for k in range(3):
        assert torch.equal(peer_rgb[k], rgb) and torch.equal(peer_a[k], alpha)
    assert torch.equal(peer_x[0], xp) and torch.equal(peer_x[1], xp)
    assert (peer_x[2] == -1.0).all()
    # a shard writes only its own rays, into the peers too (same offsets)
    pr = torch.full((V, 3, H, W), -1.0, device="cuda")
    api.dmv3d_render_views(t, intr, c2w, H, W, mlp, samples_per_ray=24, engine=engine,
                           ray_range=(2 * H * W, 4 * H * W), peers={"rgb": [pr.data_ptr()]})
    assert torch.equal(pr[2:], rgb[2:]) and (pr[:2] == -1.0).all()


@pytest.mark.parametrize("engine,dtype,T,P", [("tcgen05", "bf16", 16, 3), ("tcgen05", "bf16", 8, 2),
                                              ("simt", "f32", 16, 3)])
def test_interleaved_tiles_union_is_the_full_step(engine, dtype, T, P):
    """SURVEY §8e interleaved ray tiles: rank r writes exactly the pixels of tiles
    tau = r mod P (others untouched), and the union over ranks is the one-GPU step
    bitwise (tiles are whole 4x4 patches, so the TC tile footprint is unchanged)."""
    from paper_2605_18052_b200 import dist as pdist
    from paper_2605_18052_b200 import schedule
    tp = wl.blob_triplane(12, 32, seed=2)
    m = wl.blob_mlp(32, 64, 4, seed=3)
    if dtype == "bf16":
        tp, m = wl.round_to_bf16(tp), wl.bf16_mlp(m)
    H, W = 37, 29
    cams = wl.concat_cameras(wl.input_cameras(H, W, 2), wl.novel_cameras(H, W, 2, seed=4))
    t, intr, c2w, mlp = dev_workload(wl.Workload("tiles", tp, cams, m, 24, dtype))
    ab = schedule.cosine_alpha_bar()
    x_t = torch.from_numpy(wl.gaussian((2, 3, H, W), 4)).cuda()
    xp, rgb, alpha = api.dmv3d_render_ddim_step(t, intr, c2w, H, W, mlp, ab, 980, 960, x_t,
                                                samples_per_ray=24, engine=engine, term_eps=1e-4)
    owner = torch.tensor([[[pdist.tile_owner(v, i, j, H, W, T, P) for j in range(W)]
                           for i in range(H)] for v in range(4)], device="cuda")
    u_xp, u_rgb, u_a = torch.zeros_like(xp), torch.zeros_like(rgb), torch.zeros_like(alpha)
    for r in range(P):
        sx = torch.full_like(xp, float("nan"))
        sr = torch.full_like(rgb, float("nan"))
        sa = torch.full_like(alpha, float("nan"))
        api.dmv3d_render_ddim_step(t, intr, c2w, H, W, mlp, ab, 980, 960, x_t, x_prev=sx, rgb=sr,
                                   alpha=sa, samples_per_ray=24, engine=engine, term_eps=1e-4,
                                   tiles=(T, r, P))
        mine = owner == r
        assert not torch.isnan(sa[mine]).any() and torch.isnan(sa[~mine]).all()
        u_a[mine] = sa[mine]
        u_rgb[mine.unsqueeze(1).expand_as(rgb)] = sr[mine.unsqueeze(1).expand_as(rgb)]
        m2 = mine[:2].unsqueeze(1).expand_as(xp)
        u_xp[m2] = sx[m2]
    assert torch.equal(u_a, alpha) and torch.equal(u_rgb, rgb) and torch.equal(u_xp, xp)


@pytest.mark.parametrize("engine,dtype", [("tcgen05", "bf16"), ("simt", "f32")])
def test_tiles_with_peer_stores(engine, dtype):
    """tiles-p2p: a rank's render epilogue stores exactly its tiles' pixels into every
    peer buffer at the same offsets (peers emulated by local buffers on one GPU)."""
    from paper_2605_18052_b200 import dist as pdist
    tp = wl.blob_triplane(12, 32, seed=2)
    m = wl.blob_mlp(32, 64, 4, seed=3)
    if dtype == "bf16":
        tp, m = wl.round_to_bf16(tp), wl.bf16_mlp(m)
    H, W, T, P = 21, 18, 8, 3
    cams = wl.concat_cameras(wl.input_cameras(H, W, 2), wl.novel_cameras(H, W, 1, seed=4))
    t, intr, c2w, mlp = dev_workload(wl.Workload("tp2p", tp, cams, m, 16, dtype))
    rgb, alpha = api.dmv3d_render_views(t, intr, c2w, H, W, mlp, samples_per_ray=16, engine=engine)
    owner = torch.tensor([[[pdist.tile_owner(v, i, j, H, W, T, P) for j in range(W)]
                           for i in range(H)] for v in range(3)], device="cuda")
    for r in range(P):
        pr = [torch.full_like(rgb, -7.0) for _ in range(2)]
        pa = [torch.full_like(alpha, -7.0) for _ in range(2)]
        api.dmv3d_render_views(t, intr, c2w, H, W, mlp, samples_per_ray=16, engine=engine,
                               tiles=(T, r, P), peers={"rgb": [x.data_ptr() for x in pr],
                                                       "alpha": [x.data_ptr() for x in pa]})
        mine = owner == r
        for k in range(2):
            assert torch.equal(pa[k][mine], alpha[mine]) and (pa[k][~mine] == -7.0).all()
            m3 = mine.unsqueeze(1).expand_as(rgb)
            assert torch.equal(pr[k][m3], rgb[m3]) and (pr[k][~m3] == -7.0).all()


@pytest.mark.parametrize("engine,dtype", [("simt", "f32"), ("tcgen05", "bf16")])
def test_tiles_packed_all_gather_is_the_one_gpu_step(engine, dtype):
    """The interleaved-tile split merged by an all-gather of packed tiles: P emulated ranks
    render their tiles (fused DDIM, eta = 1 with z, a keep-mask) and dmv3d_tiles_pack
    copies them into their blocks, stacked rank by rank as the all-gather would;
    dmv3d_tiles_unpack scatters them back: bitwise the one-GPU step, on a ragged image
    (edge tiles) -- and through dist.denoise_step_tile_sharded in one process (world 1)."""
    from paper_2605_18052_b200 import dist as pdist
    tp = wl.blob_triplane(12, 32, seed=2)
    m = wl.blob_mlp(32, 64, 4, seed=3)
    if dtype == "bf16":
        tp, m = wl.round_to_bf16(tp), wl.bf16_mlp(m)
    H, W, T, P, DV = 21, 18, 8, 3, 2
    cams = wl.concat_cameras(wl.input_cameras(H, W, 2), wl.novel_cameras(H, W, 2, seed=4))
    t, intr, c2w, mlp = dev_workload(wl.Workload("tpk", tp, cams, m, 16, dtype))
    ab = schedule.cosine_alpha_bar()
    x_t = torch.from_numpy(wl.gaussian((DV, 3, H, W), 4)).cuda()
    z = torch.from_numpy(wl.gaussian((DV, 3, H, W), 5)).cuda()
    kw = dict(samples_per_ray=16, engine=engine, eta=1.0, z=z, keep_mask=[0, 1], term_eps=1e-4)
    xp, rgb, alpha = api.dmv3d_render_ddim_step(t, intr, c2w, H, W, mlp, ab, 500, 480, x_t, **kw)
    nmax = api.tiles_per_rank(4, H, W, T, P)
    g_rgb = torch.full((P * nmax, 3, T, T), -7.0, device="cuda")
    g_a = torch.full((P * nmax, T, T), -7.0, device="cuda")
    g_x = torch.full((P * nmax, 3, T, T), -7.0, device="cuda")
    for r in range(P):
        sx, sr, sa = torch.empty_like(xp), torch.empty_like(rgb), torch.empty_like(alpha)
        api.dmv3d_render_ddim_step(t, intr, c2w, H, W, mlp, ab, 500, 480, x_t, x_prev=sx, rgb=sr,
                                   alpha=sa, tiles=(T, r, P), **kw)
        b = slice(r * nmax, (r + 1) * nmax)
        api.dmv3d_tiles_pack(intr, c2w, H, W, T, r, P, sr, sa, sx, g_rgb[b], g_a[b], g_x[b], DV)
    urgb, ualpha = torch.full_like(rgb, -9.0), torch.full_like(alpha, -9.0)
    uxp = torch.full_like(xp, -9.0)
    api.dmv3d_tiles_unpack(intr, c2w, H, W, T, P, g_rgb, g_a, g_x, urgb, ualpha, uxp, DV)
    assert torch.equal(urgb, rgb) and torch.equal(ualpha, alpha) and torch.equal(uxp, xp)
    xp1, rgb1, alpha1 = pdist.denoise_step_tile_sharded(t, intr, c2w, H, W, mlp, ab, 500, 480, x_t, DV,
                                                        tile=T, **kw)
    assert torch.equal(rgb1, rgb) and torch.equal(alpha1, alpha) and torch.equal(xp1, xp)
