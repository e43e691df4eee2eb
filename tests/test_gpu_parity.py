"""GPU parity: the CUDA engine (through the C ABI) against the FP64 CPU oracle
on the same seeded inputs.

Bars (BASELINE.json north star):
  * integer binning (tile lists, brick lists, visible sets): bit-exact
  * projections and volumes: relative L2 <= 1e-4 (fp32 engine vs fp64 oracle)
  * gradients: relative L2 <= 1e-3 per parameter array
"""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import oracle as O  # noqa: E402
from tests._helpers import rel_l2  # noqa: E402

IMG_TOL = 1e-4
GRAD_TOL = 1e-3


@pytest.fixture(scope="module")
def eng():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2405_20693_b200 as P
    return P.Engine(0)


def to_engine(P, oc: "O.Cloud"):
    """Engine cloud holding the fp32 rounding of the oracle cloud; the oracle is
    re-based on exactly those fp32 values so both see identical parameters."""
    f32 = [np.asarray(a, dtype=np.float32) for a in (oc.rho_raw, oc.pos, oc.scale_raw, oc.rot)]
    ec = P.GaussianCloud(oc.s_min, *f32)
    ocf = O.Cloud.from_arrays(oc.s_min, *[a.astype(np.float64) for a in f32])
    return ec, ocf


def oscan(res, w=None):
    return O.ScannerConfig(detector_res_px=(res, w or res)) if w is None else O.ScannerConfig(detector_res_px=(w, res))


def escan(P, res, h=None):
    return P.ScannerConfig(detector_res_px=(res, h or res))


def oopts(P, o):
    return O.RasterOptions(mode=o.mode, lowpass_eps_px=o.lowpass_eps_px, dilation_compensation=o.dilation_compensation,
                           freeze_jacobian=o.freeze_jacobian, cull_mahalanobis=o.cull_mahalanobis)


def grads_to_np(g):
    return [t.detach().cpu().numpy().astype(np.float64) for t in g.tensors()]


def check_grads(eg, og, tol=GRAD_TOL, what=""):
    names = ("rho_raw", "pos", "scale_raw", "rot")
    for name, a, b in zip(names, grads_to_np(eg), (og.rho_raw, og.pos, og.scale_raw, og.rot)):
        e = rel_l2(a, b)
        assert e <= tol, f"{what} grad {name}: rel L2 {e:.3e} > {tol}"


# ---------------------------------------------------------------------- binning (bit-exact)
SCENES = [
    # (seed, count, pos_radius, smin, smax, res)
    (7, 300, 0.85, 0.02, 0.06, 129),
    (21, 2000, 0.85, 0.02, 0.06, 128),   # rasterizer_bench.cpp:14-16 cloud
    (5, 500, 0.5, 0.005, 0.3, 256),
    (9, 200, 0.9, 0.001, 0.02, 100),     # tiny footprints, partial tiles
]


@pytest.mark.parametrize("scene", SCENES)
def test_tile_lists_bit_exact(eng, scene):
    import paper_2405_20693_b200 as P
    seed, count, pr, smin, smax, res = scene
    oc = O.random_cloud(O.Rng(seed), count, pr, smin, smax)
    ec, oc = to_engine(P, oc)
    thetas = [0.37, 1.3, 2.9, 4.4, 6.0]
    fwd = eng.render(ec, escan(P, res), thetas)
    for v, th in enumerate(thetas):
        r = O.render(oc, O.test_scanner(res), th)
        off_o, idx_o = r.tile_lists()
        off_e, idx_e = fwd.tile_lists(v)
        np.testing.assert_array_equal(off_e, off_o)
        np.testing.assert_array_equal(idx_e, idx_o)


def test_tile_lists_cfg1_cloud(eng):
    import paper_2405_20693_b200 as P
    from paper_2405_20693_b200 import scenes
    ca = scenes.make_cloud(1)
    oc = O.Cloud.from_arrays(ca.s_min, *ca.as_float64())
    ec, oc = to_engine(P, oc)
    thetas = O.full_circle_angles(25)[::6]
    fwd = eng.render(ec, escan(P, 128), thetas)
    for v, th in enumerate(thetas):
        r = O.render(oc, O.test_scanner(128), th)
        off_o, idx_o = r.tile_lists()
        off_e, idx_e = fwd.tile_lists(v)
        np.testing.assert_array_equal(off_e, off_o)
        np.testing.assert_array_equal(idx_e, idx_o)


def test_project_kernels_fp64(eng):
    import paper_2405_20693_b200 as P
    oc = O.random_cloud(O.Rng(41), 400, 0.9, 0.01, 0.3)
    ec, oc = to_engine(P, oc)
    for mode in (0, 1):
        opts = P.RasterOptions(mode=mode)
        vis, rec = eng.project_kernels(ec, escan(P, 128), 0.7, opts)
        for i in range(oc.m):
            pg = O.project_kernel(oc, i, O.test_scanner(128), 0.7, oopts(P, opts))
            assert vis[i] == (pg is not None)
            if pg is None:
                continue
            ref = np.array([*pg["center"], pg["cov"][0, 0], pg["cov"][0, 1], pg["cov"][1, 1], pg["conic"][0, 0],
                            pg["conic"][0, 1], pg["conic"][1, 1], pg["amplitude"], pg["mu"], pg["depth"]])
            np.testing.assert_allclose(rec[i], ref, rtol=1e-10, atol=1e-12)


def test_mu_isotropic_kat(eng):  # test_rasterizer.cpp:33-44 through the engine
    import paper_2405_20693_b200 as P
    rng = np.random.default_rng(41)
    for i in range(20):
        s = 0.02 + 0.05 * i / 20.0
        oc = O.kernels_to_cloud(2e-4, [1.3], [rng.uniform(-0.6, 0.6, 3)], [[s, s, s]], [[1, 0, 0, 0]])
        ec, _ = to_engine(P, oc)
        sf = float(np.float32(np.log(s - 2e-4)))
        s_eff = 2e-4 + math.exp(sf)
        vis, rec = eng.project_kernels(ec, escan(P, 128), 0.7)
        assert vis[0]
        assert rec[0, 9] == pytest.approx(s_eff * math.sqrt(2 * math.pi), rel=1e-10)


# ---------------------------------------------------------------------- forward images
OPTS = [
    dict(),
    dict(mode=1),
    dict(lowpass_eps_px=0.0),
    dict(dilation_compensation=False),
    dict(cull_mahalanobis=4.0),
]


@pytest.mark.parametrize("kw", OPTS)
def test_render_forward(eng, kw):
    import paper_2405_20693_b200 as P
    oc = O.random_cloud(O.Rng(21), 2000, 0.85, 0.02, 0.06)
    ec, oc = to_engine(P, oc)
    opts = P.RasterOptions(**kw)
    thetas = [0.37, 2.0, 5.1]
    fwd = eng.render(ec, escan(P, 129), thetas, opts)
    imgs = fwd.images.cpu().numpy()
    for v, th in enumerate(thetas):
        ref = O.render(oc, O.test_scanner(129), th, oopts(P, opts)).image
        assert rel_l2(imgs[v], ref) <= IMG_TOL


def test_render_empty_and_central_value(eng):  # test_rasterizer.cpp:75-89
    import paper_2405_20693_b200 as P
    ec = P.GaussianCloud(2e-4, np.zeros(0), np.zeros(0), np.zeros(0), np.zeros(0))
    img = eng.render(ec, escan(P, 128), 0.3).image
    assert torch.count_nonzero(img).item() == 0
    oc = O.kernels_to_cloud(2e-4, [1.0], [[0, 0, 0]], [[1.0, 1.0, 1.0]], [[1, 0, 0, 0]])
    ec, _ = to_engine(P, oc)
    img = eng.render(ec, escan(P, 128), 0.0).image.cpu().numpy()
    assert img[64, 64] == pytest.approx(math.sqrt(2 * math.pi), rel=0.01)


# ---------------------------------------------------------------------- backward
@pytest.mark.parametrize("kw", OPTS + [dict(freeze_jacobian=True)])
def test_render_backward(eng, kw):
    import paper_2405_20693_b200 as P
    oc = O.random_cloud(O.Rng(22), 1500, 0.85, 0.02, 0.08)
    ec, oc = to_engine(P, oc)
    opts = P.RasterOptions(**kw)
    oo = oopts(P, opts)
    thetas = [0.37, 3.3]
    res = 129
    rng = np.random.default_rng(2)
    up = rng.uniform(-1, 1, (len(thetas), res, res)).astype(np.float32)
    fwd = eng.render(ec, escan(P, res), thetas, opts)
    g = P.CloudGrads(ec.size())
    eng.render_backward(ec, fwd, torch.from_numpy(up).cuda(), g, accumulate_stats=True)
    og = O.Grads.zeros(oc.m)
    ost = O.Stats.zeros(oc.m)
    for v, th in enumerate(thetas):
        r = O.render(oc, O.test_scanner(res), th, oo)
        O.render_backward(oc, O.test_scanner(res), th, r, up[v].astype(np.float64), og, oo, ost)
    check_grads(g, og, what=str(kw))
    assert np.array_equal(ec.grad_count.cpu().numpy(), ost.grad_count)
    assert rel_l2(ec.grad2d_norm_accum.cpu().numpy(), ost.grad2d_norm_accum) <= GRAD_TOL
    assert rel_l2(ec.grad3d_accum.cpu().numpy(), ost.grad3d_accum) <= GRAD_TOL


def test_render_backward_cfg1(eng):
    import paper_2405_20693_b200 as P
    from paper_2405_20693_b200 import scenes
    ca = scenes.make_cloud(1)
    oc = O.Cloud.from_arrays(ca.s_min, *ca.as_float64())
    ec, oc = to_engine(P, oc)
    thetas = O.full_circle_angles(25)[:3]
    rng = np.random.default_rng(2)
    up = rng.uniform(-1, 1, (3, 128, 128)).astype(np.float32)
    fwd = eng.render(ec, escan(P, 128), thetas)
    imgs = fwd.images.cpu().numpy()
    g = P.CloudGrads(ec.size())
    eng.render_backward(ec, fwd, torch.from_numpy(up).cuda(), g)
    og = O.Grads.zeros(oc.m)
    for v, th in enumerate(thetas):
        r = O.render(oc, O.test_scanner(128), th)
        assert rel_l2(imgs[v], r.image) <= IMG_TOL
        O.render_backward(oc, O.test_scanner(128), th, r, up[v].astype(np.float64), og)
    check_grads(g, og, what="cfg1")


def test_zero_upstream_and_accumulate(eng):  # test_rasterizer.cpp:226-239 + CloudGrads += semantics
    import paper_2405_20693_b200 as P
    oc = O.random_cloud(O.Rng(61), 50)
    ec, oc = to_engine(P, oc)
    fwd = eng.render(ec, escan(P, 32), 0.3)
    g = P.CloudGrads(ec.size())
    eng.render_backward(ec, fwd, torch.zeros(32, 32, device="cuda"), g)
    assert torch.count_nonzero(g.flat()).item() == 0
    up = torch.rand(32, 32, device="cuda") - 0.5
    eng.render_backward(ec, fwd, up, g)
    first = g.flat().clone()
    eng.render_backward(ec, fwd, up, g)
    assert torch.allclose(g.flat(), 2 * first, rtol=1e-6, atol=1e-12)
    with pytest.raises(P.DimMismatch):
        eng.render_backward(ec, fwd, torch.zeros(16, 16, device="cuda"), g)


def test_batched_views_equal_single_views(eng):
    import paper_2405_20693_b200 as P
    oc = O.random_cloud(O.Rng(3), 800, 0.8, 0.02, 0.1)
    ec, _ = to_engine(P, oc)
    thetas = [0.1, 1.0, 2.5, 4.0]
    up = torch.rand(4, 96, 96, device="cuda") - 0.5
    fwd = eng.render(ec, escan(P, 96), thetas)
    gb = P.CloudGrads(ec.size())
    eng.render_backward(ec, fwd, up, gb)
    gs = P.CloudGrads(ec.size())
    for v, th in enumerate(thetas):
        f1 = eng.render(ec, escan(P, 96), th)
        assert torch.equal(f1.image, fwd.images[v])  # same kernels, same order: identical bits
        eng.render_backward(ec, f1, up[v], gs)
    assert rel_l2(gb.flat().cpu().numpy(), gs.flat().cpu().numpy()) < 1e-6


def test_host_entry_points(eng):
    """sct_render_fwd_host / sct_render_bwd_host (host buffers) == device path."""
    import ctypes as C
    import paper_2405_20693_b200 as P
    from paper_2405_20693_b200 import _capi
    oc = O.random_cloud(O.Rng(8), 600, 0.8, 0.02, 0.1)
    ec, _ = to_engine(P, oc)
    host = {k: np.ascontiguousarray(v, dtype=np.float32) for k, v in ec.host_arrays().items()}
    cl = _capi.sct_cloud()
    cl.m = ec.size()
    cl.s_min_mm = ec.s_min
    for k in ("rho_raw", "pos", "scale_raw", "rot"):
        setattr(cl, k, host[k].ctypes.data)
    sc = escan(P, 64)._c()
    op = P.RasterOptions()._c()
    th = (C.c_double * 2)(0.5, 2.0)
    imgs = np.zeros((2, 64, 64), dtype=np.float32)
    st = C.c_void_p()
    L = _capi.load()
    assert L.sct_render_fwd_host(eng._h, C.byref(cl), C.byref(sc), th, 2, C.byref(op), imgs.ctypes.data,
                                 C.byref(st)) == 0
    dev = eng.render(ec, escan(P, 64), [0.5, 2.0])
    np.testing.assert_array_equal(imgs, dev.images.cpu().numpy())
    up = (np.random.default_rng(0).uniform(-1, 1, (2, 64, 64))).astype(np.float32)
    gh = {k: np.zeros_like(host[k]) for k in host}
    g = _capi.sct_grads()
    for k in gh:
        setattr(g, k, gh[k].ctypes.data)
    assert L.sct_render_bwd_host(eng._h, st, C.byref(cl), up.ctypes.data, C.byref(g), None) == 0
    L.sct_fwd_free(st)
    gd = P.CloudGrads(ec.size())
    eng.render_backward(ec, dev, torch.from_numpy(up).cuda(), gd)
    for k, t in zip(("rho_raw", "pos", "scale_raw", "rot"), gd.tensors()):
        np.testing.assert_array_equal(gh[k], t.cpu().numpy())


# ---------------------------------------------------------------------- voxelizer
GRIDS = [
    ((16, 16, 16), (-1, -1, -1), (1, 1, 1)),
    ((24, 20, 13), (-0.9, -1.1, -0.7), (1.05, 0.95, 1.2)),  # non-multiple of 8, off-centre
    ((32, 32, 32), (-1, -1, -1), (1, 1, 1)),
]


@pytest.mark.parametrize("g", GRIDS)
def test_voxel_bins_and_volume(eng, g):
    import paper_2405_20693_b200 as P
    dims, lo, hi = g
    oc = O.random_cloud(O.Rng(71), 300, 0.9, 0.02, 0.15)
    ec, oc = to_engine(P, oc)
    og = O.grid_for_extent(lo, hi, dims)
    eg = P.GridSpec(og.dims, og.origin_mm, og.spacing_mm)
    off_o, idx_o = O.voxel_bins(oc, og)
    off_e, idx_e = eng.voxel_bins(ec, eg)
    np.testing.assert_array_equal(off_e, off_o)
    np.testing.assert_array_equal(idx_e, idx_o)
    vol = eng.voxelize(ec, eg).cpu().numpy()
    ref = O.voxelize(oc, og)
    assert rel_l2(vol, ref) <= IMG_TOL
    up = np.random.default_rng(3).uniform(-1, 1, og.shape_zyx).astype(np.float32)
    gr = P.CloudGrads(ec.size())
    eng.voxelize_backward(ec, eg, torch.from_numpy(up).cuda(), gr)
    ogr = O.Grads.zeros(oc.m)
    O.voxelize_backward(oc, og, up.astype(np.float64), ogr)
    check_grads(gr, ogr, what=f"voxel {dims}")


def test_voxel_cfg1(eng):
    import paper_2405_20693_b200 as P
    from paper_2405_20693_b200 import scenes
    ca = scenes.make_cloud(1)
    oc = O.Cloud.from_arrays(ca.s_min, *ca.as_float64())
    ec, oc = to_engine(P, oc)
    og = O.grid_for_extent((-1, -1, -1), (1, 1, 1), (64, 64, 64))
    eg = P.GridSpec(og.dims, og.origin_mm, og.spacing_mm)
    off_o, idx_o = O.voxel_bins(oc, og)
    off_e, idx_e = eng.voxel_bins(ec, eg)
    np.testing.assert_array_equal(off_e, off_o)
    np.testing.assert_array_equal(idx_e, idx_o)
    assert rel_l2(eng.voxelize(ec, eg).cpu().numpy(), O.voxelize(oc, og)) <= IMG_TOL


def test_voxel_slabs_compose(eng):
    """z-slab sharding: union of slab volumes == full volume (bit-exact) and
    the sum of slab gradients == full gradient."""
    import paper_2405_20693_b200 as P
    oc = O.random_cloud(O.Rng(5), 400, 0.9, 0.02, 0.2)
    ec, _ = to_engine(P, oc)
    eg = P.grid_for_extent((-1, -1, -1), (1, 1, 1), (40, 40, 40))
    full = eng.voxelize(ec, eg)
    parts = torch.zeros_like(full)
    for zb in [(0, 2), (2, 3), (3, 5)]:
        eng.voxelize(ec, eg, z_bricks=zb, out=parts)
    assert torch.equal(parts, full)
    up = torch.rand(eg.shape_zyx, device="cuda") - 0.5
    gf = P.CloudGrads(ec.size())
    eng.voxelize_backward(ec, eg, up, gf)
    gs = P.CloudGrads(ec.size())
    for zb in [(0, 2), (2, 3), (3, 5)]:
        eng.voxelize_backward(ec, eg, up, gs, z_bricks=zb)
    assert rel_l2(gs.flat().cpu().numpy(), gf.flat().cpu().numpy()) < 1e-5


def test_voxel_kats(eng):  # test_voxelizer.cpp:11-30,109-137
    import paper_2405_20693_b200 as P
    eg = P.grid_for_extent((-1, -1, -1), (1, 1, 1), (16, 16, 16))
    c = eg.voxel_center(5, 9, 12)
    oc = O.kernels_to_cloud(2e-4, [0.42], [c], [[0.1, 0.1, 0.1]], [[1, 0, 0, 0]])
    ec, _ = to_engine(P, oc)
    rho32 = float(np.log1p(np.exp(np.float32(oc.rho_raw[0]))))
    assert eng.voxelize(ec, eg)[12, 9, 5].item() == pytest.approx(rho32, rel=1e-5)
    gz = P.CloudGrads(1)
    eng.voxelize_backward(ec, eg, torch.zeros(16, 16, 16, device="cuda"), gz)
    assert torch.count_nonzero(gz.flat()).item() == 0


# ---------------------------------------------------------------------- TV / Adam / losses
def test_tv3d(eng):
    rng = np.random.default_rng(107)
    for shape in [(6, 6, 6), (32, 32, 32), (5, 9, 7)]:
        v = rng.uniform(0, 1, shape)
        val_o, g_o = O.tv3d_loss(v)
        val, g = eng.tv3d_loss(torch.from_numpy(v.astype(np.float32)).cuda(), lam=0.05)
        assert val.item() == pytest.approx(val_o, rel=1e-5)
        assert rel_l2(g.cpu().numpy(), 0.05 * g_o) <= 1e-6
    v = np.full((8, 8, 8), 0.37, dtype=np.float32)
    val, g = eng.tv3d_loss(torch.from_numpy(v).cuda())
    assert val.item() == 0.0 and torch.count_nonzero(g).item() == 0


def test_adam(eng):
    import paper_2405_20693_b200 as P
    oc = O.random_cloud(O.Rng(3), 257)
    ec, oc = to_engine(P, oc)
    rng = np.random.default_rng(4)
    m = oc.m
    params = {k: getattr(oc, k).copy() for k in ("pos", "rho_raw", "scale_raw", "rot")}
    mo = {k: np.zeros_like(v) for k, v in params.items()}
    vo = {k: np.zeros_like(v) for k, v in params.items()}
    lrs = [2e-4, 1e-2, 5e-3, 1e-3]
    for t in range(1, 4):
        g = P.CloudGrads(m)
        gh = {}
        for k, tt in zip(("rho_raw", "pos", "scale_raw", "rot"), g.tensors()):
            a = rng.standard_normal(tt.numel()).astype(np.float32)
            tt.copy_(torch.from_numpy(a))
            gh[k] = a.astype(np.float64)
        eng.adam_step(ec, g, t, lrs)
        for k, lr in zip(("pos", "rho_raw", "scale_raw", "rot"), lrs):
            O.adam_step(params[k], mo[k], vo[k], gh[k], lr, t)
        q = params["rot"].reshape(-1, 4)
        q /= np.sqrt((q * q).sum(1, keepdims=True))
    for k in ("pos", "rho_raw", "scale_raw", "rot"):
        np.testing.assert_allclose(getattr(ec, k).cpu().numpy(), params[k], rtol=1e-5, atol=1e-6)


def test_photometric_loss(eng):
    rng = np.random.default_rng(103)
    r = rng.uniform(0, 2, (2, 40, 33)).astype(np.float32)
    m = rng.uniform(0, 1, (2, 40, 33)).astype(np.float32)
    vals, dL = eng.photometric_loss(torch.from_numpy(r).cuda(), torch.from_numpy(m).cuda(), render_scale=0.5,
                                    lambda_ssim=0.25, grad_scale=0.5)
    vals = vals.cpu().numpy()
    dL = dL.cpu().numpy()
    for i in range(2):
        rn = r[i].astype(np.float64) * 0.5
        l1, g1 = O.l1_loss(rn, m[i].astype(np.float64))
        ds, g2 = O.dssim_loss(rn, m[i].astype(np.float64))
        assert vals[i, 0] == pytest.approx(l1, rel=1e-5)
        assert vals[i, 1] == pytest.approx(ds, rel=1e-4, abs=1e-6)
        assert rel_l2(dL[i], (g1 + 0.25 * g2) * 0.5) <= 1e-4


def test_render_backward_atomic_mode():
    """Parallel-atomic reduction mode against the oracle."""
    import paper_2405_20693_b200 as P
    eng_a = P.Engine(0, deterministic=False)
    oc = O.random_cloud(O.Rng(22), 1500, 0.85, 0.02, 0.08)
    ec, oc = to_engine(P, oc)
    thetas = [0.37, 3.3]
    up = np.random.default_rng(2).uniform(-1, 1, (2, 129, 129)).astype(np.float32)
    fwd = eng_a.render(ec, escan(P, 129), thetas)
    g = P.CloudGrads(ec.size())
    eng_a.render_backward(ec, fwd, torch.from_numpy(up).cuda(), g, accumulate_stats=True)
    og = O.Grads.zeros(oc.m)
    for v, th in enumerate(thetas):
        r = O.render(oc, O.test_scanner(129), th)
        O.render_backward(oc, O.test_scanner(129), th, r, up[v].astype(np.float64), og)
    check_grads(g, og, what="atomic")


@pytest.mark.parametrize("unit_kb", [None, "96"])
def test_host_entry_points_units(eng, monkeypatch, unit_kb):
    """Many-view host-buffer calls (one composite / one K4 over all views, the
    D2H / H2D copies of view units overlapped through device flags) == device path."""
    import ctypes as C
    import paper_2405_20693_b200 as P
    from paper_2405_20693_b200 import _capi
    if unit_kb:
        monkeypatch.setenv("SCT_UNIT_KB", unit_kb)  # 64 KB views: ~1.5 views per unit
    oc = O.random_cloud(O.Rng(9), 3000, 0.8, 0.02, 0.1)
    ec, _ = to_engine(P, oc)
    host = {k: np.ascontiguousarray(v, dtype=np.float32) for k, v in ec.host_arrays().items()}
    cl = _capi.sct_cloud()
    cl.m = ec.size()
    cl.s_min_mm = ec.s_min
    for k in ("rho_raw", "pos", "scale_raw", "rot"):
        setattr(cl, k, host[k].ctypes.data)
    V, R = 37, 128
    thetas = [2 * np.pi * i / V for i in range(V)]
    sc = escan(P, R)._c()
    op = P.RasterOptions()._c()
    th = (C.c_double * V)(*thetas)
    imgs = np.zeros((V, R, R), dtype=np.float32)
    st = C.c_void_p()
    L = _capi.load()
    for rep in range(2):  # second call: next epoch on the same flags
        assert L.sct_render_fwd_host(eng._h, C.byref(cl), C.byref(sc), th, V, C.byref(op), imgs.ctypes.data,
                                     C.byref(st)) == 0, L.sct_last_error()
        dev = eng.render(ec, escan(P, R), thetas)
        np.testing.assert_array_equal(imgs, dev.images.cpu().numpy())
        up = (np.random.default_rng(rep).uniform(-1, 1, (V, R, R))).astype(np.float32)
        gh = {k: np.zeros_like(host[k]) for k in host}
        g = _capi.sct_grads()
        for k in gh:
            setattr(g, k, gh[k].ctypes.data)
        assert L.sct_render_bwd_host(eng._h, st, C.byref(cl), up.ctypes.data, C.byref(g), None) == 0, \
            L.sct_last_error()
        L.sct_fwd_free(st)
        gd = P.CloudGrads(ec.size())
        eng.render_backward(ec, dev, torch.from_numpy(up).cuda(), gd)
        for k, t in zip(("rho_raw", "pos", "scale_raw", "rot"), gd.tensors()):
            np.testing.assert_array_equal(gh[k], t.cpu().numpy())


def test_binning_paths_agree():
    """The counting-scatter binning (default) and the emit + radix-sort path
    (SCT_BIN=sort, kept for tile tables beyond shared memory) give identical
    (view, tile) lists; both are checked bit-exact against the oracle above."""
    import json
    import os
    import subprocess
    import sys
    code = r'''
import json, sys, numpy as np
sys.path.insert(0, ".")
import paper_2405_20693_b200 as P
from oracle import oracle as O
oc = O.random_cloud(O.Rng(5), 3000, 0.8, 0.005, 0.2)
f32 = [np.asarray(a, dtype=np.float32) for a in (oc.rho_raw, oc.pos, oc.scale_raw, oc.rot)]
eng = P.Engine(0)
fwd = eng.render(P.GaussianCloud(oc.s_min, *f32), P.ScannerConfig(detector_res_px=(200, 136)), [0.1, 1.7, 3.3])
out = [[a.tolist() for a in fwd.tile_lists(v)] for v in range(3)]
print(json.dumps(out))
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for mode in ("scatter", "sort"):
        env = dict(os.environ, SCT_BIN=mode)
        p = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True,
                           timeout=300)
        assert p.returncode == 0, p.stderr[-2000:]
        res[mode] = json.loads(p.stdout.strip().splitlines()[-1])
    assert res["scatter"] == res["sort"]


def test_list_schedules_agree():
    """K3/K4 process the (view, tile) lists in a longest-first order built by
    one of three sorts by list count (one-CTA block radix sort up to 8 192
    lists, a two-pass multi-CTA counting sort beyond — the 8-rank shards and
    cfg3 —, or the device-wide radix sort, SCT_ORDER_MID=0) and cut into K3 work
    items by a one-CTA or a multi-CTA scan. The schedule must not change a bit
    of the images or the (deterministic-mode) gradients: 40 views at 256^2 =
    10 240 lists, run with each path forced."""
    import os
    import subprocess
    import sys
    code = r'''
import sys, hashlib, numpy as np, torch
sys.path.insert(0, ".")
import paper_2405_20693_b200 as P
from oracle import oracle as O
oc = O.random_cloud(O.Rng(11), 2000, 0.8, 0.005, 0.12)
f32 = [np.asarray(a, dtype=np.float32) for a in (oc.rho_raw, oc.pos, oc.scale_raw, oc.rot)]
cloud = P.GaussianCloud(oc.s_min, *f32)
eng = P.Engine(0)
th = [2 * np.pi * i / 40 for i in range(40)]
fwd = eng.render(cloud, P.ScannerConfig(detector_res_px=(256, 256)), th)
g = torch.Generator().manual_seed(4)
up = (torch.rand(40, 256, 256, generator=g) - 0.5).cuda()
gr = P.CloudGrads(cloud.size())
eng.render_backward(cloud, fwd, up, gr)
h = hashlib.sha256(fwd.images.cpu().numpy().tobytes() + gr.flat().cpu().numpy().tobytes()).hexdigest()
print(h, float(fwd.images.abs().sum()))
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    for name, env in (("mid", {}), ("device_sort", {"SCT_ORDER_MID": "0"}),
                      ("one_cta_items", {"SCT_K3_SMALL": "16384"}), ("cub_items", {"SCT_K3_TWOPASS": "0"})):
        p = subprocess.run([sys.executable, "-c", code], cwd=root, env=dict(os.environ, **env), capture_output=True,
                           text=True, timeout=300)
        assert p.returncode == 0, p.stderr[-2000:]
        out[name] = p.stdout.strip().splitlines()[-1].split()
    assert float(out["mid"][1]) > 0
    assert out["mid"][0] == out["device_sort"][0] == out["one_cta_items"][0] == out["cub_items"][0], out


def test_dependent_launch_changes_no_bit():
    """Programmatic dependent launch (every engine kernel; SCT_PDL=0 disables
    it) only overlaps a kernel's launch with its predecessor's tail: images,
    deterministic gradients and a sync-free native train step are bitwise the
    same with and without it."""
    import os
    import subprocess
    import sys
    code = r'''
import sys, hashlib, numpy as np, torch
sys.path.insert(0, ".")
import paper_2405_20693_b200 as P
from oracle import oracle as O
oc = O.random_cloud(O.Rng(12), 3000, 0.8, 0.005, 0.12)
f32 = [np.asarray(a, dtype=np.float32) for a in (oc.rho_raw, oc.pos, oc.scale_raw, oc.rot)]
cloud = P.GaussianCloud(oc.s_min, *f32)
eng = P.Engine(0)
eng.set_capacity(2000000, 2000000)
th = [2 * np.pi * i / 12 for i in range(12)]
fwd = eng.render(cloud, P.ScannerConfig(detector_res_px=(192, 160)), th)
g = torch.Generator().manual_seed(5)
up = (torch.rand(12, 160, 192, generator=g) - 0.5).cuda()
gr = P.CloudGrads(cloud.size())
eng.render_backward(cloud, fwd, up, gr)
grid = P.grid_for_extent((-1, -1, -1), (1, 1, 1), (40, 40, 40))
vol = eng.voxelize(cloud, grid)
vg = P.CloudGrads(cloud.size())
eng.voxelize_backward(cloud, grid, (torch.rand(grid.shape_zyx, generator=g) - 0.5).cuda(), vg)
torch.cuda.synchronize()
assert not eng.take_overflow()
blob = b"".join(t.cpu().numpy().tobytes() for t in (fwd.images, gr.flat(), vol, vg.flat()))
print(hashlib.sha256(blob).hexdigest())
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    for pdl in ("1", "0"):
        p = subprocess.run([sys.executable, "-c", code], cwd=root, env=dict(os.environ, SCT_PDL=pdl),
                           capture_output=True, text=True, timeout=300)
        assert p.returncode == 0, p.stderr[-2000:]
        out[pdl] = p.stdout.strip().splitlines()[-1]
    assert out["1"] == out["0"], out
