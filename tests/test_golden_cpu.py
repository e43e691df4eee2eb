"""The FP64 restatement against the committed golden fixtures (tests/golden/,
outputs of the reference's own sources, oracle/_ref): tile/brick lists
bit-exact, gradients to 1e-12, and the fixtures load through the engine's
readers of the reference container formats. CPU only."""
import numpy as np
import pytest

from oracle import oracle as O
from tests import _golden as G
from tests._helpers import rel_l2


def _cloud(case="rectified"):
    s_min, *arrs = G.cloud_arrays(case)
    return O.Cloud.from_arrays(s_min, *[a.astype(np.float64) for a in arrs])


@pytest.mark.parametrize("name", G.RASTER_SETS)
def test_oracle_reproduces_raster_golden(name):
    man, imgs, dL, z = G.raster(name)
    c = _cloud(name)
    cfg = O.ScannerConfig(detector_res_px=tuple(man["raster"]["res"]))
    opts = O.RasterOptions(**man["option_sets"][name])
    g, st = O.Grads.zeros(c.m), O.Stats.zeros(c.m)
    for v, th in enumerate(man["raster"]["thetas"]):
        r = O.render(c, cfg, th, opts)
        off, idx = r.tile_lists()
        np.testing.assert_array_equal(off, z[f"offsets{v}"])
        np.testing.assert_array_equal(idx, z[f"idx{v}"])
        np.testing.assert_allclose(r.image, imgs[v], rtol=1e-6, atol=1e-7)  # fp32 container
        O.render_backward(c, cfg, th, r, dL[v].astype(np.float64), g, opts, st)
    for k in ("rho_raw", "pos", "scale_raw", "rot"):
        assert rel_l2(getattr(g, k), z["g_" + k]) < 1e-12, k
    np.testing.assert_array_equal(st.grad_count, z["grad_count"])
    assert rel_l2(st.grad2d_norm_accum, z["grad2d_norm_accum"]) < 1e-12


def test_oracle_reproduces_voxel_golden():
    grid, vol, dL, z = G.voxel()
    c = _cloud()
    og = O.GridSpec(grid.dims, grid.origin_mm, grid.spacing_mm)
    off, idx = O.voxel_bins(c, og)
    np.testing.assert_array_equal(off, z["offsets"])
    np.testing.assert_array_equal(idx, z["idx"])
    np.testing.assert_allclose(O.voxelize(c, og), vol, rtol=1e-6, atol=1e-7)
    g = O.Grads.zeros(c.m)
    O.voxelize_backward(c, og, dL.astype(np.float64), g)
    for k in ("rho_raw", "pos", "scale_raw", "rot"):
        assert rel_l2(getattr(g, k), z["g_" + k]) < 1e-12, k
