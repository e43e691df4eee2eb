"""GPU parity for sub-pixel kernels ("narrow-kernel parity hole").

The reference evaluates exp(-1/2 d^T Q d) exactly for any footprint
(rasterizer.cpp:151) and supports lowpass_eps_px = 0 (rasterizer.cpp:44-50;
test_rasterizer.cpp:49,186). With a small low-pass the projected sigma drops
below ~0.25 px, where K3/K4's exp2 ratio recurrence would lose a run's peak;
those chunks take the direct per-pixel evaluation (raster.cu kRun4MaxA_*).

Clouds with projected sigma 0.03-0.3 px at the cfg3 geometry, eps in {0, 0.1},
both reduction modes, on 129^2 (partial tiles) and 512^2 detectors, against
the FP64 oracle: tile lists bit-exact, images <= 1e-4, gradients <= 1e-3.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import oracle as O  # noqa: E402
from tests._helpers import rel_l2  # noqa: E402

IMG_TOL, GRAD_TOL = 1e-4, 1e-3


def _px_sigma_mm(res):
    # detector pixel at the detector plane, demagnified to the rotation axis (L_SO / L_SD)
    return 5.6 / res * 8.0 / 12.0


@pytest.mark.parametrize("res", [129, 512])
@pytest.mark.parametrize("eps", [0.0, 0.1])
@pytest.mark.parametrize("deterministic", [True, False])
def test_narrow_kernels_match_oracle(res, eps, deterministic):
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    import paper_2405_20693_b200 as P
    px = _px_sigma_mm(res)
    m = 1500 if res == 512 else 600
    oc = O.random_cloud(O.Rng(97 + res), m, 0.8, 0.03 * px, 0.3 * px, s_min=1e-5)
    f32 = [np.asarray(a, dtype=np.float32) for a in (oc.rho_raw, oc.pos, oc.scale_raw, oc.rot)]
    ec = P.GaussianCloud(oc.s_min, *f32)
    oc = O.Cloud.from_arrays(oc.s_min, *[a.astype(np.float64) for a in f32])
    eng = P.Engine(0, deterministic=deterministic)
    thetas = [0.37, 2.2]
    opts = P.RasterOptions(lowpass_eps_px=eps)
    oopt = O.RasterOptions(lowpass_eps_px=eps)
    ocfg = O.test_scanner(res)
    fwd = eng.render(ec, P.ScannerConfig(detector_res_px=(res, res)), thetas, opts)
    imgs = fwd.images.cpu().numpy()
    up = np.random.default_rng(5).uniform(-1, 1, (len(thetas), res, res)).astype(np.float32)
    og, ost = O.Grads.zeros(oc.m), O.Stats.zeros(oc.m)
    for v, th in enumerate(thetas):
        r = O.render(oc, ocfg, th, oopt)
        off_o, idx_o = r.tile_lists()
        off_e, idx_e = fwd.tile_lists(v)
        np.testing.assert_array_equal(off_e, off_o)
        np.testing.assert_array_equal(idx_e, idx_o)
        e = rel_l2(imgs[v], r.image)
        assert e <= IMG_TOL, f"view {v} image rel L2 {e:.3e}"
        O.render_backward(oc, ocfg, th, r, up[v].astype(np.float64), og, oopt, ost)
    g = P.CloudGrads(ec.size())
    eng.render_backward(ec, fwd, torch.from_numpy(up).cuda(), g, accumulate_stats=True)
    torch.cuda.synchronize()
    for k in ("rho_raw", "pos", "scale_raw", "rot"):
        e = rel_l2(getattr(g, k).cpu().numpy().astype(np.float64), getattr(og, k))
        assert e <= GRAD_TOL, f"grad {k} rel L2 {e:.3e}"
    np.testing.assert_array_equal(ec.grad_count.cpu().numpy(), ost.grad_count)
    fwd.free()


def test_narrow_kernel_peak_not_lost():
    """A single kernel with sigma 0.1 px centred on a pixel: the image holds its
    peak (the recurrence alone would flush it to zero)."""
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    import paper_2405_20693_b200 as P
    res = 512
    s = 0.1 * _px_sigma_mm(res)
    for th in (0.0, 0.5):
        # centre on the ray through pixel (300, 200)'s centre, at the rotation axis depth
        o, d = O.pixel_ray(O.test_scanner(res), th, 300, 200)
        p = o + 8.0 * d
        oc = O.kernels_to_cloud(1e-5, [1.0], [p], [[s, s, s]], [[1.0, 0.0, 0.0, 0.0]])
        f32 = [np.asarray(a, dtype=np.float32) for a in (oc.rho_raw, oc.pos, oc.scale_raw, oc.rot)]
        ec = P.GaussianCloud(oc.s_min, *f32)
        oc = O.Cloud.from_arrays(oc.s_min, *[a.astype(np.float64) for a in f32])
        for eps in (0.0, 0.1):
            fwd = P.Engine(0).render(ec, P.ScannerConfig(detector_res_px=(res, res)), [th],
                                     P.RasterOptions(lowpass_eps_px=eps))
            img = fwd.images.cpu().numpy()[0]
            ref = O.render(oc, O.test_scanner(res), th, O.RasterOptions(lowpass_eps_px=eps)).image
            assert ref.max() > 0.5 * ref.sum()  # one dominant pixel
            assert rel_l2(img, ref) <= IMG_TOL
            fwd.free()
