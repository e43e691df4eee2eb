"""voxelize(keep_state=True) + voxelize_backward(state=...) share one binning;
results must equal the re-binning entry points (the reference's semantics)
bitwise, on the full grid and on z-slabs."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import oracle as O  # noqa: E402


@pytest.mark.parametrize("zb", [None, (1, 3)])
def test_voxel_state_equals_rebinning(zb):
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    import paper_2405_20693_b200 as P
    oc = O.random_cloud(O.Rng(8), 600, 0.9, 0.02, 0.2)
    c = P.GaussianCloud(oc.s_min, *[np.asarray(a, np.float32) for a in (oc.rho_raw, oc.pos, oc.scale_raw, oc.rot)])
    eng = P.Engine(0)
    g = P.grid_for_extent((-1, -1, -1), (1, 1, 1), (36, 30, 28))
    up = torch.rand(g.shape_zyx, device="cuda") - 0.5
    v1 = eng.voxelize(c, g, z_bricks=zb)
    g1 = P.CloudGrads(c.size())
    eng.voxelize_backward(c, g, up, g1, z_bricks=zb)
    v2, st = eng.voxelize(c, g, z_bricks=zb, keep_state=True)
    g2 = P.CloudGrads(c.size())
    eng.voxelize_backward(c, g, up, g2, z_bricks=zb, state=st)
    st.free()
    torch.cuda.synchronize()
    assert torch.equal(v1, v2)
    assert torch.equal(g1.buffer, g2.buffer)
