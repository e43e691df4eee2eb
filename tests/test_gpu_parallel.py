"""Parallel-beam geometry (extension named by the north star; no reference code)
through the C-ABI against the oracle's parallel-beam restatement: tile lists
bit-exact, images <= 1e-4, gradients and statistics <= 1e-3 in both modes and
both reduction orders, FP64 projection export, and the quadrature projector."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import oracle as O  # noqa: E402
from tests._helpers import rel_l2  # noqa: E402


def _P():
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    import paper_2405_20693_b200 as P
    return P


@pytest.mark.parametrize("mode,deterministic", [(0, True), (1, True), (0, False)])
def test_parallel_render_parity(mode, deterministic):
    P = _P()
    eng = P.Engine(0, deterministic=deterministic)
    oc = O.random_cloud(O.Rng(77), 600, 0.8, 0.01, 0.12)
    f32 = [np.asarray(a, np.float32) for a in (oc.rho_raw, oc.pos, oc.scale_raw, oc.rot)]
    oc = O.Cloud.from_arrays(oc.s_min, *[a.astype(np.float64) for a in f32])
    ec = P.GaussianCloud(oc.s_min, *f32)
    w, h = 130, 100
    ocfg = O.ScannerConfig(detector_res_px=(w, h), parallel_beam=True)
    ecfg = P.ScannerConfig(detector_res_px=(w, h), parallel_beam=True)
    thetas = [0.2, 1.9, 4.0]
    oo = O.RasterOptions(mode=mode)
    eo = P.RasterOptions(mode=mode)
    fwd = eng.render(ec, ecfg, thetas, eo)
    imgs = fwd.images.cpu().numpy()
    rng = O.Rng(3)
    ups = np.stack([O.random_image(rng, w, h, -1, 1) for _ in thetas]).astype(np.float32)
    og, ost = O.Grads.zeros(oc.m), O.Stats.zeros(oc.m)
    for v, th in enumerate(thetas):
        r = O.render(oc, ocfg, th, oo)
        off_o, idx_o = r.tile_lists()
        off_e, idx_e = fwd.tile_lists(v)
        np.testing.assert_array_equal(off_e, off_o)
        np.testing.assert_array_equal(idx_e, idx_o)
        assert rel_l2(imgs[v], r.image) <= 1e-4
        O.render_backward(oc, ocfg, th, r, ups[v].astype(np.float64), og, oo, ost)
    g = P.CloudGrads(ec.size())
    eng.render_backward(ec, fwd, torch.from_numpy(ups).cuda(), g, accumulate_stats=True)
    torch.cuda.synchronize()
    for k in ("rho_raw", "pos", "scale_raw", "rot"):
        assert rel_l2(getattr(g, k).cpu().numpy(), getattr(og, k)) <= 1e-3, k
    np.testing.assert_array_equal(ec.grad_count.cpu().numpy(), ost.grad_count)
    assert rel_l2(ec.grad2d_norm_accum.cpu().numpy(), ost.grad2d_norm_accum) <= 1e-3
    fwd.free()


def test_parallel_project_export_and_projector():
    P = _P()
    eng = P.Engine(0)
    oc = O.random_cloud(O.Rng(91), 50, 0.7, 0.02, 0.2)
    ec = P.GaussianCloud(oc.s_min, *[np.asarray(a, np.float32) for a in (oc.rho_raw, oc.pos, oc.scale_raw, oc.rot)])
    oc = O.Cloud.from_arrays(oc.s_min, *[np.asarray(a, np.float32).astype(np.float64)
                                         for a in (oc.rho_raw, oc.pos, oc.scale_raw, oc.rot)])
    ecfg = P.ScannerConfig(detector_res_px=(64, 48), parallel_beam=True)
    ocfg = O.ScannerConfig(detector_res_px=(64, 48), parallel_beam=True)
    vis, rec = eng.project_kernels(ec, ecfg, 0.9)
    for i in range(oc.m):
        r = O.project_kernel(oc, i, ocfg, 0.9)
        assert vis[i] == (r is not None)
        if r is not None:
            np.testing.assert_allclose(rec[i, :2], r["center"], rtol=1e-12)
            assert rec[i, 8] == pytest.approx(r["amplitude"], rel=1e-10)
            assert rec[i, 10] == pytest.approx(r["depth"], rel=1e-12)
    from oracle import fixtures as FX
    from paper_2405_20693_b200 import simulate as S
    ph, grid = S.phantom_shepp_logan_3d((32, 32, 32))
    got = S.project_volume(ph, grid, ecfg, [0.0, 0.7], 0.03).cpu().numpy()
    og = O.GridSpec(grid.dims, grid.origin_mm, grid.spacing_mm)
    for v, th in enumerate([0.0, 0.7]):
        assert rel_l2(got[v], FX.project_volume(ph.cpu().numpy(), og, ocfg, th, 0.03)) <= 1e-6
    with pytest.raises(P.ConfigError):
        S.fdk_reconstruct(S.project_volume(ph, grid, ecfg, [0.0, 1.0], 0.03), ecfg, [0.0, 1.0], grid)
