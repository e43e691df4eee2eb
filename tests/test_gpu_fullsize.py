"""Parity at BASELINE.json's full sizes (the bench workloads, not reduced
scenes): cfg3 (100k Gaussians, 512² detector, 75 views) and cfg4 (200k
Gaussians, 256³ grid), through the C ABI against the FP64 CPU oracle.

The oracle runs a bounded sample of each workload (two views; a z-slab) so the
test stays within seconds; the engine runs the full batch, and the sampled
views are compared exactly where the bar is exact (tile / brick lists) and at
the stated tolerances elsewhere. Size-independent properties cover the rest:
the full 75-view gradient equals the sum of per-view gradients, and the
voxelizer's slab volume equals the corresponding part of the full volume.
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


@pytest.fixture(scope="module")
def cfg3():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    sys.path.insert(0, ROOT)
    import bench
    import paper_2405_20693_b200 as P
    w, ca, thetas, vol = bench.make_workload()
    f32 = [np.asarray(a, dtype=np.float32) for a in (ca.rho_raw, ca.pos, ca.scale_raw, ca.rot)]
    ec = P.GaussianCloud(ca.s_min, *f32)
    oc = O.Cloud.from_arrays(ca.s_min, *[a.astype(np.float64) for a in f32])
    return P, w, ec, oc, thetas, vol


def test_cfg3_lists_images_grads(cfg3):
    P, w, ec, oc, thetas, _ = cfg3
    eng = P.Engine(0)
    res = w.res
    up = np.random.default_rng(2).uniform(-1, 1, (len(thetas), res, res)).astype(np.float32)
    fwd = eng.render(ec, P.ScannerConfig(detector_res_px=(res, res)), thetas)
    imgs = fwd.images.cpu().numpy()
    g = P.CloudGrads(ec.size())
    eng.render_backward(ec, fwd, torch.from_numpy(up).cuda(), g)
    og_views = O.Grads.zeros(oc.m)
    for v in VIEWS:
        r = O.render(oc, O.test_scanner(res), thetas[v])
        off_o, idx_o = r.tile_lists()
        off_e, idx_e = fwd.tile_lists(v)
        np.testing.assert_array_equal(off_e, off_o)  # 1024 tiles, ~400k (tile, kernel) pairs per view
        np.testing.assert_array_equal(idx_e, idx_o)
        assert rel_l2(imgs[v], r.image) <= IMG_TOL
        O.render_backward(oc, O.test_scanner(res), thetas[v], r, up[v].astype(np.float64), og_views)
    # the sampled views' gradient, from the engine, against the oracle
    gv = P.CloudGrads(ec.size())
    sub = eng.render(ec, P.ScannerConfig(detector_res_px=(res, res)), [thetas[v] for v in VIEWS])
    eng.render_backward(ec, sub, torch.from_numpy(up[list(VIEWS)]).cuda(), gv)
    for a, b in zip(gv.tensors(), (og_views.rho_raw, og_views.pos, og_views.scale_raw, og_views.rot)):
        assert rel_l2(a.cpu().numpy().astype(np.float64), b) <= GRAD_TOL
    # size-independent: the 75-view batch gradient is the sum of per-view gradients
    gs = P.CloudGrads(ec.size())
    for v0 in range(0, len(thetas), 25):
        vs = list(range(v0, min(v0 + 25, len(thetas))))
        part = eng.render(ec, P.ScannerConfig(detector_res_px=(res, res)), [thetas[v] for v in vs])
        eng.render_backward(ec, part, torch.from_numpy(up[vs]).cuda(), gs)
    torch.cuda.synchronize()
    assert rel_l2(g.flat().cpu().numpy(), gs.flat().cpu().numpy()) < 1e-5


def test_cfg4_bins_and_volume_slab(cfg3):
    P, _, _, _, _, vol = cfg3
    from paper_2405_20693_b200 import scenes
    ca = scenes.make_cloud(4, vol=vol)
    f32 = [np.asarray(a, dtype=np.float32) for a in (ca.rho_raw, ca.pos, ca.scale_raw, ca.rot)]
    ec = P.GaussianCloud(ca.s_min, *f32)
    oc = O.Cloud.from_arrays(ca.s_min, *[a.astype(np.float64) for a in f32])
    eng = P.Engine(0)
    n = scenes.CONFIGS[4].n_vox
    grid = P.grid_for_extent((-1, -1, -1), (1, 1, 1), (n, n, n))
    full = eng.voxelize(ec, grid).cpu().numpy()
    # a 2-brick-layer central slab through the oracle: 16 voxel layers
    z0, nz = n // 2 - 8, 16
    og = O.GridSpec((n, n, nz), (grid.origin_mm[0], grid.origin_mm[1], grid.origin_mm[2] + z0 * grid.spacing_mm[2]),
                    tuple(grid.spacing_mm))
    ref = O.voxelize(oc, og)
    assert rel_l2(full[z0:z0 + nz], ref) <= IMG_TOL
    # brick lists of the slab grid, bit-exact
    eg = P.GridSpec((n, n, nz), og.origin_mm, og.spacing_mm)
    off_e, idx_e = eng.voxel_bins(ec, eg)
    off_o, idx_o = O.voxel_bins(oc, og)
    np.testing.assert_array_equal(off_e, off_o)
    np.testing.assert_array_equal(idx_e, idx_o)
