"""Device fixture generation (csrc/fixtures.cu) against the
FP64 oracle restatement (oracle/fixtures_oracle.cpp): phantom bit-exact,
quadrature projections and FDK volumes <= 1e-6 relative L2 (FP64 on both sides,
fp32 storage), nearest-neighbour distances exact, init clouds equal (same
std::mt19937_64 stream), plus the reference's own KATs on the device path."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import fixtures as FX  # noqa: E402
from oracle import oracle as O  # noqa: E402
from tests._helpers import rel_l2  # noqa: E402


def _S():
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    import paper_2405_20693_b200 as P
    from paper_2405_20693_b200 import simulate as S
    return P, S


def _ogrid(g):
    return O.GridSpec(g.dims, g.origin_mm, g.spacing_mm)


@pytest.mark.parametrize("dims,lo,hi", [((64, 64, 64), (-1, -1, -1), (1, 1, 1)),
                                        ((40, 33, 17), (-1.0, -0.8, -0.6), (0.9, 1.0, 0.7))])
def test_phantom_bit_exact(dims, lo, hi):
    P, S = _S()
    vol, grid = S.phantom_shepp_logan_3d(dims, lo, hi)
    np.testing.assert_array_equal(vol.cpu().numpy(), FX.phantom(dims, lo, hi))
    with pytest.raises(P.ConfigError):
        S.phantom_shepp_logan_3d((8, 64, 64))


def test_project_volume_matches_oracle_and_kats():
    P, S = _S()
    ph, grid = S.phantom_shepp_logan_3d((32, 32, 32))
    cfg = P.ScannerConfig(detector_res_px=(129, 97))
    thetas = [0.0, 0.3, 2.2]
    imgs = S.project_volume(ph, grid, cfg, thetas, 0.03).cpu().numpy()
    ocfg = O.ScannerConfig(detector_res_px=(129, 97))
    for v, th in enumerate(thetas):
        ref = FX.project_volume(ph.cpu().numpy(), _ogrid(grid), ocfg, th, 0.03)
        assert rel_l2(imgs[v], ref) <= 1e-6
    # test_simulator.cpp:65-80: uniform volume chord, zero volume
    sq = P.ScannerConfig(detector_res_px=(129, 129))
    g32 = P.grid_for_extent((-1, -1, -1), (1, 1, 1), (32, 32, 32))
    img = S.project_volume(torch.full((32, 32, 32), 0.8, device="cuda"), g32, sq, 0.0, 0.01).cpu().numpy()
    assert img[64, 64] == pytest.approx(1.6, rel=1e-3)
    g16 = P.grid_for_extent((-1, -1, -1), (1, 1, 1), (16, 16, 16))
    assert not S.project_volume(torch.zeros((16, 16, 16), device="cuda"), g16, sq, 0.7, 0.05).any()
    with pytest.raises(P.ConfigError):
        S.project_volume(ph, grid, cfg, 0.3, 0.0)


@pytest.mark.parametrize("window", [0, 1, 2])
def test_fdk_matches_oracle(window):
    P, S = _S()
    ph, grid = S.phantom_shepp_logan_3d((32, 32, 32))
    cfg = P.ScannerConfig(detector_res_px=(48, 40))
    thetas = O.full_circle_angles(24)
    proj = S.project_volume(ph, grid, cfg, thetas, 0.5 * grid.spacing_mm[0])
    vol = S.fdk_reconstruct(proj, cfg, thetas, grid, window).cpu().numpy()
    ref = FX.fdk(proj.cpu().numpy(), O.ScannerConfig(detector_res_px=(48, 40)), thetas, _ogrid(grid), window)
    assert rel_l2(vol, ref) <= 1e-6
    with pytest.raises(P.DataError):
        S.fdk_reconstruct(proj[:1], cfg, thetas[:1], grid)


def test_fdk_kats():  # test_fdk.cpp:23-78 on the device
    P, S = _S()
    cfg = P.ScannerConfig(detector_res_px=(32, 32))
    g16 = P.grid_for_extent((-1, -1, -1), (1, 1, 1), (16, 16, 16))
    th = O.full_circle_angles(10)
    assert not S.fdk_reconstruct(torch.zeros((10, 32, 32), device="cuda"), cfg, th, g16).any()
    ph, g64 = S.phantom_shepp_logan_3d((64, 64, 64))
    c64 = P.ScannerConfig(detector_res_px=(64, 64))
    th100 = O.full_circle_angles(100)
    dense = S.project_volume(ph, g64, c64, th100, 0.5 * g64.spacing_mm[0])
    rec = S.fdk_reconstruct(dense, c64, th100, g64)
    mse = float(((rec.clamp(0, 1) - ph) ** 2).mean())
    p_dense = 10 * np.log10(1 / mse)
    assert p_dense >= 18.5  # see tests/test_oracle_fixtures.py for the reference's 25 dB claim
    sparse = S.fdk_reconstruct(dense[::4], c64, th100[::4], g64)
    assert 10 * np.log10(1 / float(((sparse.clamp(0, 1) - ph) ** 2).mean())) < p_dense


def test_nn_distances_exact():
    P, S = _S()
    rng = np.random.default_rng(5)
    pts = rng.uniform(-1, 1, (3001, 3))
    pts[7] = pts[11]  # a duplicate point has distance 0
    got = S.nearest_neighbor_distances(torch.from_numpy(pts)).cpu().numpy()
    np.testing.assert_array_equal(got, FX.nn_distances(pts))
    assert got[7] == 0.0


def test_sample_init_cloud_matches_oracle():
    P, S = _S()
    ph, grid = S.phantom_shepp_logan_3d((48, 48, 48))
    cl = S.sample_init_cloud(ph, grid, 3000, seed=13)
    oc = FX.sample_init_cloud(O.Rng(13), ph.cpu().numpy(), _ogrid(grid), 3000)
    np.testing.assert_array_equal(cl.pos.cpu().numpy(), oc.pos.astype(np.float32))
    np.testing.assert_allclose(cl.scale_raw.cpu().numpy(), oc.scale_raw, rtol=2e-7, atol=2e-7)
    np.testing.assert_allclose(cl.rho_raw.cpu().numpy(), oc.rho_raw, rtol=2e-7, atol=2e-7)
    np.testing.assert_array_equal(cl.rot.cpu().numpy(), oc.rot.astype(np.float32))
    with pytest.raises(P.DataError):  # TooFewOccupiedVoxels
        S.sample_init_cloud(torch.zeros_like(ph), grid, 2)


def test_pipeline_phantom_to_trainable_cloud():
    """simulate (noisy) -> FDK -> init -> render: the reference's train() inputs, all on device."""
    P, S = _S()
    ph, grid = S.phantom_shepp_logan_3d((64, 64, 64))
    cfg = P.ScannerConfig(detector_res_px=(96, 96))
    th = O.full_circle_angles(40)
    proj = S.simulate_projections(ph, grid, cfg, th, 0.5 * grid.spacing_mm[0], S.NoiseParams(seed=3))
    assert proj.shape == (40, 96, 96) and torch.isfinite(proj).all()
    vol = S.fdk_reconstruct(proj, cfg, th, grid)
    cloud = S.sample_init_cloud(vol, grid, 5000, seed=0)
    eng = P.default_engine()
    img = eng.render(cloud, cfg, th[:2]).images
    assert torch.isfinite(img).all() and float(img.max()) > 0
