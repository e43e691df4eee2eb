"""The engine (through the C-ABI) against the committed golden fixtures
(tests/golden/, outputs of the reference's own sources — oracle/_ref — in the
reference container formats, written by its io.cpp):
tile lists and voxel brick lists bit-exact, images / volumes <= 1e-4 rel L2,
gradients and adaptive statistics <= 1e-3 (BASELINE.json parity bars), in both
reduction modes."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from tests import _golden as G  # noqa: E402
from tests._helpers import rel_l2  # noqa: E402

IMG_TOL, GRAD_TOL = 1e-4, 1e-3


def _setup(case="rectified"):
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    import paper_2405_20693_b200 as P
    s_min, *arrs = G.cloud_arrays(case)
    return P, P.GaussianCloud(s_min, *arrs)


@pytest.mark.parametrize("deterministic", [True, False])
@pytest.mark.parametrize("name", G.RASTER_SETS)
def test_engine_matches_raster_golden(name, deterministic):
    P, c = _setup(name)
    eng = P.Engine(0, deterministic=deterministic)
    man, imgs, dL, z = G.raster(name)
    w, h = man["raster"]["res"]
    opts = P.RasterOptions(**man["option_sets"][name])
    fwd = eng.render(c, P.ScannerConfig(detector_res_px=(w, h)), man["raster"]["thetas"], opts)
    out = fwd.images.cpu().numpy()
    for v in range(len(man["raster"]["thetas"])):
        off, idx = fwd.tile_lists(v)
        np.testing.assert_array_equal(off, z[f"offsets{v}"])
        np.testing.assert_array_equal(idx, z[f"idx{v}"])
        assert rel_l2(out[v], imgs[v]) <= IMG_TOL
    g = P.CloudGrads(c.size())
    eng.render_backward(c, fwd, torch.from_numpy(dL).cuda(), g, accumulate_stats=True)
    torch.cuda.synchronize()
    for k in ("rho_raw", "pos", "scale_raw", "rot"):
        assert rel_l2(getattr(g, k).cpu().numpy(), z["g_" + k]) <= GRAD_TOL, k
    np.testing.assert_array_equal(c.grad_count.cpu().numpy(), z["grad_count"])
    assert rel_l2(c.grad2d_norm_accum.cpu().numpy(), z["grad2d_norm_accum"]) <= GRAD_TOL
    assert rel_l2(c.grad3d_accum.cpu().numpy(), z["grad3d_accum"]) <= GRAD_TOL
    fwd.free()


def test_engine_matches_voxel_golden():
    P, c = _setup()
    eng = P.Engine(0)
    grid, vol, dL, z = G.voxel()
    off, idx = eng.voxel_bins(c, grid)
    np.testing.assert_array_equal(off, z["offsets"])
    np.testing.assert_array_equal(idx, z["idx"])
    assert rel_l2(eng.voxelize(c, grid).cpu().numpy(), vol) <= IMG_TOL
    g = P.CloudGrads(c.size())
    eng.voxelize_backward(c, grid, torch.from_numpy(dL).cuda(), g)
    torch.cuda.synchronize()
    for k in ("rho_raw", "pos", "scale_raw", "rot"):
        assert rel_l2(getattr(g, k).cpu().numpy(), z["g_" + k]) <= GRAD_TOL, k
