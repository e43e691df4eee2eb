"""Parallel-beam extension of the oracle (north_star: "cone- or parallel-beam
detector planes"). The reference has no parallel-beam code or test, so this
geometry is pinned analytically (SURVEY.md §8c "parity unpinned" for the
reference): the orthographic map is affine, so the rasterised line integral is
exact — without the 0.3 px low-pass it must equal a fine ray march of the 3D
density along the parallel rays — and render_backward must pass the same
finite-difference check as the cone-beam path. CPU only."""
import numpy as np
import pytest

from oracle import oracle as O
from tests._helpers import finite_difference_check


def _par(res=128):
    return O.ScannerConfig(detector_res_px=(res, res), parallel_beam=True)


def test_parallel_pixel_rays_are_parallel():
    cfg = _par(64)
    o0, d0 = O.pixel_ray(cfg, 0.7, 3, 5)
    o1, d1 = O.pixel_ray(cfg, 0.7, 60, 41)
    np.testing.assert_allclose(d0, d1, atol=1e-15)
    # detector pixel pitch maps 1:1 to scanner millimetres (no magnification)
    oa, _ = O.pixel_ray(cfg, 0.7, 10, 10)
    ob, _ = O.pixel_ray(cfg, 0.7, 11, 10)
    assert np.linalg.norm(ob - oa) == pytest.approx(5.6 / 64, rel=1e-12)


@pytest.mark.parametrize("theta", [0.0, 1.1, 2.9])
def test_parallel_render_equals_ray_march(theta):
    cl = O.random_cloud(O.Rng(53), 3, 0.25, 0.12, 0.18)
    cfg = _par()
    exact = O.RasterOptions(lowpass_eps_px=0.0)
    img = O.render(cl, cfg, theta, exact).image
    peak = img.max()
    checked = 0
    for v in range(0, 128, 3):
        for u in range(0, 128, 3):
            if img[v, u] < 0.05 * peak:
                continue
            o, d = O.pixel_ray(cfg, theta, u, v)
            ref = O.ray_march_density(cl, o, d, 1e-3)
            assert abs(img[v, u] - ref) / ref < 1e-5
            checked += 1
    assert checked > 20
    # with the default low-pass + compensation the mass is preserved to 1e-3
    dflt = O.render(cl, cfg, theta).image
    assert abs(dflt.sum() - img.sum()) / img.sum() < 1e-3


def test_parallel_amplitude_is_the_z_integral():
    # one isotropic kernel: the exact line integral of rho exp(-|x|^2/2s^2) is rho s sqrt(2 pi)
    s, rho = 0.1, 0.7
    cl = O.kernels_to_cloud(2e-4, [rho], [[0.0, 0.0, 0.0]], [[s, s, s]], [[1, 0, 0, 0]])
    rec = O.project_kernel(cl, 0, _par(64), 0.3, O.RasterOptions(lowpass_eps_px=0.0))
    assert rec is not None
    assert rec["mu"] == pytest.approx(s * np.sqrt(2 * np.pi), rel=1e-12)
    assert rec["amplitude"] == pytest.approx(rho * s * np.sqrt(2 * np.pi), rel=1e-12)


@pytest.mark.parametrize("mode", [0, 1])
def test_parallel_render_backward_fd(mode):
    cfg = O.ScannerConfig(detector_res_px=(16, 16), parallel_beam=True)
    rng = O.Rng(59)
    for scene in range(3):
        cloud = O.random_cloud(rng, 4, 0.3, 0.1, 0.3)
        opts = O.RasterOptions(mode=mode)
        up = O.random_image(rng, 16, 16, -1.0, 1.0)
        loss = lambda c: float(np.sum(O.render(c, cfg, 0.8, opts).image * up))
        fwd = O.render(cloud, cfg, 0.8, opts)
        g = O.Grads.zeros(4)
        O.render_backward(cloud, cfg, 0.8, fwd, up, g, opts)
        err, n = finite_difference_check(cloud, g, loss)
        assert n == 44 and err < 1e-4, (scene, err)


def test_parallel_freeze_jacobian_is_a_no_op():
    cfg = _par(32)
    cl = O.random_cloud(O.Rng(61), 5)
    up = O.random_image(O.Rng(62), 32, 32, -1, 1)
    out = []
    for frozen in (False, True):
        opts = O.RasterOptions(freeze_jacobian=frozen)
        g = O.Grads.zeros(5)
        O.render_backward(cl, cfg, 0.3, O.render(cl, cfg, 0.3, opts), up, g, opts)
        out.append(g.flat())
    np.testing.assert_array_equal(out[0], out[1])


def test_parallel_projector_agrees_with_rasterizer():
    """test_simulator.cpp:184-206 in parallel-beam geometry: voxelize -> quadrature projector
    vs direct rasterisation."""
    from oracle import fixtures as FX
    cfg = O.ScannerConfig(detector_res_px=(64, 64), parallel_beam=True)
    cloud = O.random_cloud(O.Rng(113), 4, 0.25, 0.12, 0.2)
    fine = O.grid_for_extent((-1, -1, -1), (1, 1, 1), (96, 96, 96))
    vol = O.voxelize(cloud, fine).astype(np.float32)
    for theta in (0.0, np.pi / 3):
        via = FX.project_volume(vol, fine, cfg, theta, 0.01)
        # without the 0.3 px low-pass (0.026 mm in object space here, 1.5x the cone-beam
        # test's) the raster value is the exact line integral
        direct = O.render(cloud, cfg, theta, O.RasterOptions(lowpass_eps_px=0.0)).image
        peak = direct.max()
        n = 0
        for v in range(8, 56, 2):
            for u in range(8, 56, 2):
                if direct[v, u] < 0.3 * peak:
                    continue
                assert abs(direct[v, u] - via[v, u]) / direct[v, u] < 0.02
                n += 1
        assert n > 5
