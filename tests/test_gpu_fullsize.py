"""Parity at BASELINE.json's full sizes (the bench workloads, not reduced
scenes), through the C ABI against the FP64 CPU oracle:

* cfg3 (100k Gaussians, 512^2 detector, 75 views) in BOTH reduction modes —
  deterministic and the parallel-atomic mode bench.py times;
* cfg4 (200k Gaussians, 256^3 grid): brick lists, volume AND backward
  gradients on a central slab; the full-grid backward equals the sum of its
  slab backwards;
* cfg5 (1M Gaussians, 512^3 phantom, 1024^2 detector): one sampled view of the
  100 (tile lists, image, gradients), and a 512x512x136 slab of the 512^3 grid,
  whose 69,632 bricks exceed 16-bit brick keys (the uint32 key path).

The oracle runs a bounded sample of each workload (sampled views; a z-slab) so
the test stays within tens of seconds; the engine runs the full batch where it
matters, and the sampled pieces are compared exactly where the bar is exact
(tile / brick lists) and at the stated tolerances elsewhere.
"""
import os
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import oracle as O  # noqa: E402
from tests._helpers import rel_l2  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
IMG_TOL = 1e-4
GRAD_TOL = 1e-3
VIEWS = (0, 37)  # sampled views of the 75 (theta = 0 and ~pi)


def _pair(P, ca):
    f32 = [np.asarray(a, dtype=np.float32) for a in (ca.rho_raw, ca.pos, ca.scale_raw, ca.rot)]
    return P.GaussianCloud(ca.s_min, *f32), O.Cloud.from_arrays(ca.s_min, *[a.astype(np.float64) for a in f32])


@pytest.fixture(scope="module")
def cfg3():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    sys.path.insert(0, ROOT)
    import bench
    import paper_2405_20693_b200 as P
    w, ca, thetas, vol = bench.make_workload()
    ec, oc = _pair(P, ca)
    res = w.res
    up = np.random.default_rng(2).uniform(-1, 1, (len(thetas), res, res)).astype(np.float32)
    # the oracle's sampled views, computed once for both reduction modes
    og = O.Grads.zeros(oc.m)
    ref = {}
    for v in VIEWS:
        r = O.render(oc, O.test_scanner(res), thetas[v])
        ref[v] = (r.tile_lists(), r.image)
        O.render_backward(oc, O.test_scanner(res), thetas[v], r, up[v].astype(np.float64), og)
    return P, w, ec, oc, thetas, vol, up, ref, og


@pytest.mark.parametrize("deterministic", [True, False], ids=["deterministic", "atomic"])
def test_cfg3_lists_images_grads(cfg3, deterministic):
    P, w, ec, oc, thetas, _, up, ref, og = cfg3
    eng = P.Engine(0, deterministic=deterministic)
    res = w.res
    fwd = eng.render(ec, P.ScannerConfig(detector_res_px=(res, res)), thetas)
    imgs = fwd.images.cpu().numpy()
    g = P.CloudGrads(ec.size())
    eng.render_backward(ec, fwd, torch.from_numpy(up).cuda(), g)
    for v in VIEWS:
        (off_o, idx_o), img_o = ref[v]
        off_e, idx_e = fwd.tile_lists(v)
        np.testing.assert_array_equal(off_e, off_o)  # 1024 tiles, ~400k (tile, kernel) pairs per view
        np.testing.assert_array_equal(idx_e, idx_o)
        assert rel_l2(imgs[v], img_o) <= IMG_TOL
    # the sampled views' gradient, from the engine, against the oracle
    gv = P.CloudGrads(ec.size())
    sub = eng.render(ec, P.ScannerConfig(detector_res_px=(res, res)), [thetas[v] for v in VIEWS])
    eng.render_backward(ec, sub, torch.from_numpy(up[list(VIEWS)]).cuda(), gv)
    for a, b in zip(gv.tensors(), (og.rho_raw, og.pos, og.scale_raw, og.rot)):
        assert rel_l2(a.cpu().numpy().astype(np.float64), b) <= GRAD_TOL
    # size-independent: the 75-view batch gradient is the sum of per-view gradients
    gs = P.CloudGrads(ec.size())
    for v0 in range(0, len(thetas), 25):
        vs = list(range(v0, min(v0 + 25, len(thetas))))
        part = eng.render(ec, P.ScannerConfig(detector_res_px=(res, res)), [thetas[v] for v in vs])
        eng.render_backward(ec, part, torch.from_numpy(up[vs]).cuda(), gs)
    torch.cuda.synchronize()
    assert rel_l2(g.flat().cpu().numpy(), gs.flat().cpu().numpy()) < 1e-5


@pytest.fixture(scope="module")
def cfg4(cfg3):
    P, _, _, _, _, vol, *_ = cfg3
    from paper_2405_20693_b200 import scenes
    ec, oc = _pair(P, scenes.make_cloud(4, vol=vol))
    n = scenes.CONFIGS[4].n_vox
    return P, ec, oc, n


@pytest.mark.parametrize("deterministic", [True, False], ids=["deterministic", "atomic"])
def test_cfg4_bins_volume_grads_slab(cfg4, deterministic):
    P, ec, oc, n = cfg4
    eng = P.Engine(0, deterministic=deterministic)
    grid = P.grid_for_extent((-1, -1, -1), (1, 1, 1), (n, n, n))
    full = eng.voxelize(ec, grid).cpu().numpy()
    # a 2-brick-layer central slab through the oracle: 16 voxel layers
    z0, nz = n // 2 - 8, 16
    origin = (grid.origin_mm[0], grid.origin_mm[1], grid.origin_mm[2] + z0 * grid.spacing_mm[2])
    og = O.GridSpec((n, n, nz), origin, tuple(grid.spacing_mm))
    ref = O.voxelize(oc, og)
    assert rel_l2(full[z0:z0 + nz], ref) <= IMG_TOL
    eg = P.GridSpec((n, n, nz), og.origin_mm, og.spacing_mm)
    off_e, idx_e = eng.voxel_bins(ec, eg)
    off_o, idx_o = O.voxel_bins(oc, og)
    np.testing.assert_array_equal(off_e, off_o)
    np.testing.assert_array_equal(idx_e, idx_o)
    # backward gradients on the slab grid (upstream U(-1,1), seed 3)
    dl = np.random.default_rng(3).uniform(-1, 1, og.shape_zyx).astype(np.float32)
    ge = P.CloudGrads(ec.size())
    eng.voxelize_backward(ec, eg, torch.from_numpy(dl).cuda(), ge)
    go = O.Grads.zeros(oc.m)
    O.voxelize_backward(oc, og, dl.astype(np.float64), go)
    torch.cuda.synchronize()
    for a, b in zip(ge.tensors(), (go.rho_raw, go.pos, go.scale_raw, go.rot)):
        assert rel_l2(a.cpu().numpy().astype(np.float64), b) <= GRAD_TOL
    # size-independent: the full-grid backward equals the sum of its z-slab backwards
    up = torch.from_numpy(np.random.default_rng(4).uniform(-1, 1, grid.shape_zyx).astype(np.float32)).cuda()
    gf = P.CloudGrads(ec.size())
    eng.voxelize_backward(ec, grid, up, gf)
    gsum = P.CloudGrads(ec.size())
    nzb = (n + 7) // 8
    for zb in range(0, nzb, 8):
        eng.voxelize_backward(ec, grid, up, gsum, z_bricks=(zb, min(nzb, zb + 8)))
    torch.cuda.synchronize()
    assert rel_l2(gf.flat().cpu().numpy(), gsum.flat().cpu().numpy()) < 1e-5


@pytest.fixture(scope="module")
def cfg5():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2405_20693_b200 as P
    from paper_2405_20693_b200 import scenes, simulate
    w = scenes.CONFIGS[5]
    # the device fixture path (phantom + FDK-free init; parity-tested in
    # test_gpu_fixtures.py) — the host numpy path takes minutes at 512^3
    vol, grid = simulate.phantom_shepp_logan_3d((w.n_vox,) * 3)
    cl = simulate.sample_init_cloud(vol, grid, w.m, s_min_mm=2e-4, seed=0)
    raw = {k: getattr(cl, k).cpu().numpy().astype(np.float64) for k in ("rho_raw", "pos", "scale_raw", "rot")}
    rho = np.where(raw["rho_raw"] > 30.0, raw["rho_raw"], np.log1p(np.exp(np.minimum(raw["rho_raw"], 30.0))))
    scale = cl.s_min + np.exp(raw["scale_raw"].reshape(-1, 3))  # gaussian_cloud.cpp:9-28
    rho, pos, scale, rot = scenes.trained_like(rho, raw["pos"].reshape(-1, 3), scale, raw["rot"].reshape(-1, 4),
                                               cl.s_min, seed=1)
    ca = scenes._raw(cl.s_min, rho, pos, scale, rot)
    del vol
    torch.cuda.empty_cache()
    ec, oc = _pair(P, ca)
    return P, w, ec, oc


def test_cfg5_sampled_view(cfg5):
    P, w, ec, oc = cfg5
    eng = P.Engine(0, deterministic=False)
    res = w.res
    thetas = P.full_circle_angles(w.n_views)
    v = 31
    up = np.random.default_rng(9).uniform(-1, 1, (1, res, res)).astype(np.float32)
    fwd = eng.render(ec, P.ScannerConfig(detector_res_px=(res, res)), [thetas[v]])
    r = O.render(oc, O.test_scanner(res), thetas[v])
    off_o, idx_o = r.tile_lists()
    off_e, idx_e = fwd.tile_lists(0)
    np.testing.assert_array_equal(off_e, off_o)  # 4096 tiles, ~3M (tile, kernel) pairs
    np.testing.assert_array_equal(idx_e, idx_o)
    assert rel_l2(fwd.images.cpu().numpy()[0], r.image) <= IMG_TOL
    g = P.CloudGrads(ec.size())
    eng.render_backward(ec, fwd, torch.from_numpy(up).cuda(), g)
    og = O.Grads.zeros(oc.m)
    O.render_backward(oc, O.test_scanner(res), thetas[v], r, up[0].astype(np.float64), og)
    torch.cuda.synchronize()
    for a, b in zip(g.tensors(), (og.rho_raw, og.pos, og.scale_raw, og.rot)):
        assert rel_l2(a.cpu().numpy().astype(np.float64), b) <= GRAD_TOL
    fwd.free()


def test_cfg5_slab_uint32_brick_keys(cfg5):
    P, w, ec, oc = cfg5
    eng = P.Engine(0, deterministic=False)
    n = w.n_vox
    grid = P.grid_for_extent((-1, -1, -1), (1, 1, 1), (n, n, n))
    nz = 136  # 17 brick layers: 64 * 64 * 17 = 69,632 bricks > 65,536
    z0 = n // 2 - 64
    origin = (grid.origin_mm[0], grid.origin_mm[1], grid.origin_mm[2] + z0 * grid.spacing_mm[2])
    og = O.GridSpec((n, n, nz), origin, tuple(grid.spacing_mm))
    eg = P.GridSpec((n, n, nz), og.origin_mm, og.spacing_mm)
    assert (n // 8) * (n // 8) * (nz // 8) > 65536
    off_e, idx_e = eng.voxel_bins(ec, eg)
    off_o, idx_o = O.voxel_bins(oc, og)
    np.testing.assert_array_equal(off_e, off_o)
    np.testing.assert_array_equal(idx_e, idx_o)
    vol_e = eng.voxelize(ec, eg).cpu().numpy()
    assert rel_l2(vol_e, O.voxelize(oc, og)) <= IMG_TOL
    # and the slab of the full 512^3 volume (262,144 bricks) is the same volume
    full = eng.voxelize(ec, grid)
    assert rel_l2(full[z0:z0 + nz].cpu().numpy(), vol_e) <= 1e-6
