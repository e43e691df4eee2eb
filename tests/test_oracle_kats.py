"""Pins the CPU oracle (oracle/splatct_oracle.cpp) against every known-answer
and property test the reference ships for the hot path. The reference has no
golden vectors; these are its own tests re-expressed in pytest,
on the same std::mt19937_64 scenes (file:line cited per test).
Every test runs twice: against the FP64 restatement ("port") and against the
reference's own sources compiled into oracle/_ref ("reference") — the latter
shows the build shims (oracle/ref_shim/) reproduce the reference's own test
verdicts. CPU only — no GPU needed."""
import math

import numpy as np
import pytest

from oracle import oracle as O
from tests._helpers import finite_difference_check


@pytest.fixture(autouse=True, params=["port", "reference"])
def oracle_kind(request):
    if request.param == "reference" and not O.ref_available():
        pytest.skip("oracle/_ref (the compiled reference) not built")
    with O.using(request.param):
        yield request.param


def single_kernel_cloud(rho, p, s, q=(1.0, 0.0, 0.0, 0.0), s_min=2e-4):
    return O.kernels_to_cloud(s_min, [rho], [p], [s], [q])


# ----------------------------------------------------------- geometry
def test_view_transform_convention():  # test_geometry.cpp:27-47
    c = O.test_scanner()
    rot0, t0 = O.view_transform(c, 0.0)
    assert np.abs(rot0 - np.array([[0, 1, 0], [0, 0, -1], [-1, 0, 0]])).max() < 1e-15
    assert np.linalg.norm(t0 - [0, 0, 8.0]) < 1e-15
    rot90, _ = O.view_transform(c, math.pi / 2)
    assert np.abs(rot90 - np.array([[-1, 0, 0], [0, 0, -1], [0, -1, 0]])).max() < 1e-12


def test_view_transform_rigid():  # test_geometry.cpp:49-57
    c = O.test_scanner()
    for i in range(64):
        r, _ = O.view_transform(c, 2 * math.pi * i / 64 + 0.123)
        assert np.abs(r.T @ r - np.eye(3)).max() < 1e-12
        assert abs(np.linalg.det(r) - 1.0) < 1e-12


def test_pixel_ray_and_round_trip():  # test_geometry.cpp:59-103
    c = O.test_scanner(129)
    o, d = O.pixel_ray(c, 0.0, 64, 64)
    assert np.linalg.norm(o - [8.0, 0, 0]) < 1e-12
    assert np.linalg.norm(d - [-1, 0, 0]) < 1e-12
    rng = np.random.default_rng(11)
    for i in range(100):
        u, v = rng.integers(0, 129, size=2)
        theta = 2 * math.pi * i / 100
        o, d = O.pixel_ray(c, theta, int(u), int(v))
        p = o + rng.uniform(4.0, 12.0) * d
        rot, t = O.view_transform(c, theta)
        m = O.ray_space_point(c, rot @ p + t)
        assert abs(m[0] - (u + 0.5)) < 1e-6 and abs(m[1] - (v + 0.5)) < 1e-6


def test_local_jacobian():  # test_geometry.cpp:105-147
    c = O.test_scanner()
    det = O.detector_model(c)
    j = O.local_jacobian(c, [0, 0, 7.0])
    assert j[0, 0] == pytest.approx(det["fx"] / 7.0, rel=1e-14)
    assert j[0, 1] == 0.0 and j[0, 2] == 0.0 and j[1, 2] == 0.0
    rng = np.random.default_rng(3)
    for _ in range(100):
        p = np.array([rng.uniform(-1, 1), rng.uniform(-1, 1), rng.uniform(6, 10)])
        j = O.local_jacobian(c, p)
        fd = np.zeros((3, 3))
        h = 1e-5
        for k in range(3):
            hi, lo = p.copy(), p.copy()
            hi[k] += h
            lo[k] -= h
            fd[:, k] = (O.ray_space_point(c, hi) - O.ray_space_point(c, lo)) / (2 * h)
        assert np.abs(j - fd).max() / np.abs(j).max() < 1e-6
    with pytest.raises(O.OracleError):
        O.local_jacobian(c, [0, 0, 0.04])


# ----------------------------------------------------------- cloud math
def test_covariance_assembly():  # test_gaussian_cloud.cpp:13-46
    cl = single_kernel_cloud(1.0, (0, 0, 0), (1.0, 2.0, 3.0), s_min=1e-4)
    assert np.abs(O.covariance_at(cl, 0) - np.diag([1.0, 4.0, 9.0])).max() < 1e-12
    rng = O.Rng(5)
    for _ in range(20):
        q = [rng.normal() for _ in range(4)][::-1]
        cl = single_kernel_cloud(1.0, (0, 0, 0), (1.0, 2.0, 3.0), q, s_min=1e-4)
        s = O.covariance_at(cl, 0)
        assert np.linalg.det(s) == pytest.approx(36.0, rel=1e-12)
        assert np.abs(np.sort(np.linalg.eigvalsh(s)) - [1, 4, 9]).max() < 1e-9


def test_density_at():  # test_gaussian_cloud.cpp:48-70
    cl = single_kernel_cloud(0.7, (0.1, -0.2, 0.3), (0.2, 0.2, 0.2), s_min=1e-4)
    assert O.density_at(cl, [0.1, -0.2, 0.3]) == pytest.approx(0.7, rel=1e-12)
    assert O.density_at(cl, [0.3, -0.2, 0.3]) == pytest.approx(0.7 * math.exp(-0.5), rel=1e-12)


def test_covariance_chain_fd():  # test_gaussian_cloud.cpp:120-165
    rng = O.Rng(23)
    cloud = O.random_cloud(rng, 3)
    g = np.random.default_rng(0).normal(size=(3, 3))
    up = g + g.T

    def loss(c):
        return sum(float(np.sum(up * O.covariance_at(c, i))) for i in range(c.m))

    grads = O.Grads.zeros(cloud.m)
    for i in range(cloud.m):
        O.accumulate_covariance_param_grads(cloud, i, up, grads)
    fd_cloud = cloud.copy()
    worst = 0.0
    for name in ("scale_raw", "rot"):
        p = getattr(fd_cloud, name)
        a = getattr(grads, name)
        for i in range(p.size):
            s = p[i]
            h = 1e-6 * max(1.0, abs(s))
            p[i] = s + h
            u = loss(fd_cloud)
            p[i] = s - h
            d = loss(fd_cloud)
            p[i] = s
            fd = (u - d) / (2 * h)
            worst = max(worst, abs(fd - a[i]) / max(abs(fd), abs(a[i]), 1e-6))
    assert worst < 1e-5


# ----------------------------------------------------------- rasterizer
def test_mu_isotropic():  # test_rasterizer.cpp:33-44
    cfg = O.test_scanner()
    rng = np.random.default_rng(41)
    for i in range(20):
        s = 0.02 + 0.05 * i / 20.0
        cl = single_kernel_cloud(1.3, rng.uniform(-0.6, 0.6, 3), (s, s, s))
        pg = O.project_kernel(cl, 0, cfg, 0.7)
        assert pg is not None
        assert pg["mu"] == pytest.approx(s * math.sqrt(2 * math.pi), rel=1e-10)


def test_amplitude_modes_and_cull():  # test_rasterizer.cpp:46-69
    cfg = O.test_scanner()
    cl = single_kernel_cloud(0.8, (0.1, 0.0, -0.1), (0.1, 0.1, 0.1))
    rect = O.project_kernel(cl, 0, cfg, 0.7, O.RasterOptions(lowpass_eps_px=0.0))
    bias = O.project_kernel(cl, 0, cfg, 0.7, O.RasterOptions(mode=1, lowpass_eps_px=0.0))
    assert rect["amplitude"] == pytest.approx(rect["mu"] * 0.8, rel=1e-12)
    assert bias["amplitude"] == pytest.approx(0.8, rel=1e-12)
    assert bias["mu"] == pytest.approx(rect["mu"], rel=1e-12)
    cl = single_kernel_cloud(1.0, (2 * 8.0 * math.cos(0.7), 2 * 8.0 * math.sin(0.7), 0.0), (0.1, 0.1, 0.1))
    assert O.project_kernel(cl, 0, cfg, 0.7) is None


def test_render_basics():  # test_rasterizer.cpp:72-122
    cfg = O.test_scanner()
    assert np.all(O.render(O.Cloud.empty(), cfg, 0.3).image == 0.0)
    cl = single_kernel_cloud(1.0, (0, 0, 0), (1.0, 1.0, 1.0))
    img = O.render(cl, cfg, 0.0).image
    assert img[64, 64] == pytest.approx(math.sqrt(2 * math.pi), rel=0.01)
    rng = O.Rng(43)
    a = O.random_cloud(rng, 5)
    b = O.random_cloud(rng, 4)
    both = a.concat(b)
    ia, ib, iab = (O.render(c, cfg, 0.9).image for c in (a, b, both))
    assert np.abs(iab - ia - ib).max() < 1e-10
    rng = O.Rng(47)
    c = O.random_cloud(rng, 20)
    perm = np.random.default_rng(1).permutation(20)
    sh = O.Cloud(c.s_min, c.rho_raw[perm].copy(), c.pos.reshape(-1, 3)[perm].ravel().copy(),
                 c.scale_raw.reshape(-1, 3)[perm].ravel().copy(), c.rot.reshape(-1, 4)[perm].ravel().copy())
    assert np.abs(O.render(c, cfg, 1.7).image - O.render(sh, cfg, 1.7).image).max() < 1e-10


def test_view_consistency():  # test_rasterizer.cpp:124-154
    cfg = O.test_scanner(129)
    q = np.array([0.9, 0.2, -0.3, 0.1])
    cl = single_kernel_cloud(0.9, (0, 0, 0), (0.08, 0.16, 0.24), q / np.linalg.norm(q))
    rect, bias = [], []
    for th in O.full_circle_angles(12):
        pg = O.project_kernel(cl, 0, cfg, th)
        rect.append(O.render(cl, cfg, th).image[64, 64] / pg["mu"])
        bias.append(O.render(cl, cfg, th, O.RasterOptions(mode=1)).image[64, 64] / pg["mu"])
    spread = lambda v: (max(v) - min(v)) / np.mean(v)
    assert spread(rect) < 0.01
    assert all(abs(r - 0.9) / 0.9 < 0.01 for r in rect)
    assert spread(bias) > 0.10


def test_ray_march_oracle():  # test_rasterizer.cpp:156-178
    cfg = O.test_scanner()
    rng = O.Rng(53)
    cl = O.random_cloud(rng, 3, 0.25, 0.12, 0.18)
    for th in (0.0, 1.1):
        img = O.render(cl, cfg, th).image
        peak = img.max()
        checked = 0
        for v in range(0, 128, 3):
            for u in range(0, 128, 3):
                if img[v, u] < 0.2 * peak:
                    continue
                o, d = O.pixel_ray(cfg, th, u, v)
                ref = O.ray_march_density(cl, o, d, 1e-3)
                assert abs(img[v, u] - ref) / ref < 0.01
                checked += 1
        assert checked > 10


def test_lowpass_mass():  # test_rasterizer.cpp:180-192
    cfg = O.test_scanner()
    cl = single_kernel_cloud(1.0, (0.05, -0.02, 0.1), (0.175, 0.175, 0.175))
    a = O.render(cl, cfg, 0.4).image.sum()
    b = O.render(cl, cfg, 0.4, O.RasterOptions(lowpass_eps_px=0.0)).image.sum()
    assert abs(a - b) / b < 1e-3


@pytest.mark.parametrize("mode", [0, 1])
def test_render_backward_fd(mode):  # test_rasterizer.cpp:194-224 (+ acceptance criterion 1)
    cfg = O.test_scanner(16)
    rng = O.Rng(59)
    for scene in range(3):
        cloud = O.random_cloud(rng, 4, 0.3, 0.1, 0.3)
        opts = O.RasterOptions(mode=mode)
        up = O.random_image(rng, 16, 16, -1.0, 1.0)
        loss = lambda c: float(np.sum(O.render(c, cfg, 0.8, opts).image * up))
        fwd = O.render(cloud, cfg, 0.8, opts)
        assert fwd.n_visible == 4
        g = O.Grads.zeros(4)
        O.render_backward(cloud, cfg, 0.8, fwd, up, g, opts)
        err, n = finite_difference_check(cloud, g, loss)
        assert n == 44 and err < 1e-4, (scene, err)


def test_zero_upstream_and_frozen_jacobian():  # test_rasterizer.cpp:226-263
    cfg = O.test_scanner(32)
    rng = O.Rng(61)
    cl = O.random_cloud(rng, 3)
    fwd = O.render(cl, cfg, 0.3)
    g = O.Grads.zeros(3)
    O.render_backward(cl, cfg, 0.3, fwd, np.zeros((32, 32)), g)
    assert not g.flat().any()
    cfg = O.test_scanner(16)
    rng = O.Rng(67)
    cl = O.random_cloud(rng, 2, 0.3, 0.15, 0.3)
    up = O.random_image(rng, 16, 16, -1.0, 1.0)
    frozen = O.RasterOptions(freeze_jacobian=True)
    fwd = O.render(cl, cfg, 0.5, frozen)
    gf, gfull = O.Grads.zeros(2), O.Grads.zeros(2)
    O.render_backward(cl, cfg, 0.5, fwd, up, gf, frozen)
    O.render_backward(cl, cfg, 0.5, fwd, up, gfull, O.RasterOptions())
    np.testing.assert_allclose(gf.rho_raw, gfull.rho_raw, rtol=1e-12)
    assert np.abs(gf.pos - gfull.pos).max() > 0.0


def test_dim_mismatch():  # rasterizer.cpp:201-202
    cfg = O.test_scanner(16)
    cl = O.random_cloud(O.Rng(1), 2)
    fwd = O.render(cl, cfg, 0.5)
    with pytest.raises(O.DimMismatch):
        O.render_backward(cl, cfg, 0.5, fwd, np.zeros((8, 8)), O.Grads.zeros(2))


def test_tile_lists_ascending_and_cover():  # rasterizer.cpp:123-133
    cfg = O.test_scanner(129)
    cl = O.random_cloud(O.Rng(7), 300, 0.85, 0.02, 0.06)
    r = O.render(cl, cfg, 0.37)
    off, idx = r.tile_lists()
    assert off[-1] == r.n_pairs
    for t in range(len(off) - 1):
        seg = idx[off[t]:off[t + 1]]
        assert np.all(np.diff(seg) > 0)


# ----------------------------------------------------------- voxelizer
def test_voxelize_basics():  # test_voxelizer.cpp:11-30
    grid = O.grid_for_extent((-1, -1, -1), (1, 1, 1), (16, 16, 16))
    assert not O.voxelize(O.Cloud.empty(), grid).any()
    cl = single_kernel_cloud(0.42, grid.voxel_center(5, 9, 12), (0.1, 0.1, 0.1))
    assert O.voxelize(cl, grid)[12, 9, 5] == pytest.approx(0.42, rel=1e-12)


def test_voxelize_full_sum():  # test_voxelizer.cpp:32-53 (+ acceptance criterion 5)
    grid = O.grid_for_extent((-1, -1, -1), (1, 1, 1), (32, 32, 32))
    vox = grid.spacing_mm[0]
    rng = O.Rng(71)
    worst = 0.0
    for _ in range(10):
        cl = O.random_cloud(rng, 20, 0.8, 0.5 * vox, 1.4 * vox)
        vol = O.voxelize(cl, grid)
        peak = cl.rho().max()
        for z in range(0, 32, 4):
            for y in range(0, 32, 4):
                for x in range(0, 32, 4):
                    ref = O.density_at(cl, grid.voxel_center(x, y, z))
                    worst = max(worst, abs(vol[z, y, x] - ref) / peak)
    assert worst < 1e-3


def test_voxelize_linear_and_monotone():  # test_voxelizer.cpp:55-81
    grid = O.grid_for_extent((-1, -1, -1), (1, 1, 1), (16, 16, 16))
    rng = O.Rng(73)
    a = O.random_cloud(rng, 6)
    b = O.random_cloud(rng, 5)
    assert np.abs(O.voxelize(a.concat(b), grid) - O.voxelize(a, grid) - O.voxelize(b, grid)).max() < 1e-12
    grid = O.grid_for_extent((-1, -1, -1), (1, 1, 1), (24, 24, 24))
    cl = O.random_cloud(O.Rng(79), 15, 0.8, 0.05, 0.3)
    vt = O.voxelize(cl, grid)
    vl = O.voxelize(cl, grid, 5.0)
    assert np.all(vl >= vt - 1e-15)


def test_voxelize_backward_fd():  # test_voxelizer.cpp:83-107
    grid = O.grid_for_extent((-1, -1, -1), (1, 1, 1), (8, 8, 8))
    rng = O.Rng(83)
    for _ in range(3):
        cl = O.random_cloud(rng, 4, 0.4, 0.2, 0.5)
        up = O.random_image(rng, 64, 8, -1.0, 1.0).reshape(8, 8, 8)
        loss = lambda c: float(np.sum(O.voxelize(c, grid) * up))
        g = O.Grads.zeros(4)
        O.voxelize_backward(cl, grid, up, g)
        err, _ = finite_difference_check(cl, g, loss)
        assert err < 1e-4


def test_voxelize_backward_edges():  # test_voxelizer.cpp:109-137
    grid = O.grid_for_extent((-1, -1, -1), (1, 1, 1), (8, 8, 8))
    cl = O.random_cloud(O.Rng(89), 3)
    g = O.Grads.zeros(3)
    O.voxelize_backward(cl, grid, np.zeros((8, 8, 8)), g)
    assert not g.flat().any()
    up = np.zeros((8, 8, 8))
    up[5, 4, 3] = 1.0
    g = O.Grads.zeros(3)
    O.voxelize_backward(cl, grid, up, g)
    c = grid.voxel_center(3, 4, 5)
    for i in range(3):
        d = c - cl.pos[3 * i:3 * i + 3]
        w = math.exp(-0.5 * d @ np.linalg.inv(O.covariance_at(cl, i)) @ d)
        sig = 1.0 / (1.0 + math.exp(-cl.rho_raw[i]))
        assert g.rho_raw[i] / sig == pytest.approx(w, rel=1e-9)


def test_random_subvolume_spec():  # test_voxelizer.cpp:139-162
    sp = (2 / 64,) * 3
    rng = O.Rng(97)
    for _ in range(50):
        g = O.random_subvolume_spec((-1,) * 3, (1,) * 3, sp, 32, rng)
        for k in range(3):
            assert g.origin_mm[k] >= -1 and g.origin_mm[k] + 32 * sp[k] <= 1 + 1e-12
    a = O.random_subvolume_spec((-1,) * 3, (1,) * 3, sp, 16, O.Rng(123))
    b = O.random_subvolume_spec((-1,) * 3, (1,) * 3, sp, 16, O.Rng(123))
    assert a.origin_mm == b.origin_mm


# ----------------------------------------------------------- objectives / optimizer
def test_tv3d():  # test_objectives.cpp:88-127
    v = np.full((8, 8, 8), 0.37)
    val, g = O.tv3d_loss(v)
    assert val == 0.0 and not g.any()
    v = np.array([0, 1, 0, 1, 0, 1, 0, 1], dtype=np.float64).reshape(2, 2, 2)
    assert O.tv3d_loss(v)[0] == pytest.approx(1.0, rel=1e-12)
    rng = O.Rng(107)
    v = O.random_image(rng, 36, 6).reshape(6, 6, 6)
    val, g = O.tv3d_loss(v)
    worst = 0.0
    for i in range(v.size):
        f = v.reshape(-1)
        s = f[i]
        f[i] = s + 1e-7
        up = O.tv3d_loss(v)[0]
        f[i] = s - 1e-7
        dn = O.tv3d_loss(v)[0]
        f[i] = s
        worst = max(worst, abs(g.reshape(-1)[i] - (up - dn) / 2e-7))
    assert worst < 1e-6
    with pytest.raises(O.DimMismatch):
        O.tv3d_loss(np.zeros((1, 4, 4)))


def test_l1_dssim():  # test_objectives.cpp:37-86
    rng = O.Rng(101)
    a = O.random_image(rng, 16, 16)
    assert O.l1_loss(a, a)[0] == 0.0
    assert O.l1_loss(a + 0.25, a)[0] == pytest.approx(0.25, rel=1e-12)
    rng = O.Rng(103)
    a = O.random_image(rng, 16, 16)
    b = O.random_image(rng, 16, 16)
    assert O.dssim_loss(a, a)[0] == pytest.approx(0.0, abs=1e-12)
    val, g = O.dssim_loss(a, b)
    gs = np.abs(g).max()
    worst = 0.0
    for i in range(a.size):
        f = a.reshape(-1)
        s = f[i]
        f[i] = s + 1e-6
        up = O.dssim_loss(a, b)[0]
        f[i] = s - 1e-6
        dn = O.dssim_loss(a, b)[0]
        f[i] = s
        fd = (up - dn) / 2e-6
        worst = max(worst, abs(g.reshape(-1)[i] - fd) / max(abs(fd), abs(g.reshape(-1)[i]), 1e-3 * gs))
    assert worst < 1e-5
    with pytest.raises(O.DimMismatch):
        O.dssim_loss(np.zeros((8, 8)), np.zeros((8, 8)))


def test_lr_schedule():  # test_trainer.cpp:37-44
    for lr in (0.0002, 0.01, 0.005, 0.001):
        assert abs(O.lr_at(lr, 0.1, 30000, 30000) - 0.1 * lr) < 1e-12
        assert O.lr_at(lr, 0.1, 0, 30000) == pytest.approx(lr)
        assert O.lr_at(lr, 0.1, 15000, 30000) == pytest.approx(lr * math.sqrt(0.1), rel=1e-12)


def test_clone_halving_mass():  # test_trainer.cpp:213-230
    cfg = O.test_scanner(64)
    rng = O.Rng(0)
    cl = O.random_cloud(rng, 6, 0.3, 0.05, 0.2)
    before = O.render(cl, cfg, 0.7).image
    rho = cl.rho()
    half = 0.5 * rho[2]
    raw_half = O.kernels_to_cloud(cl.s_min, [half], [cl.pos[6:9]], [cl.scale()[2]], [cl.rot[8:12]])
    cloned = cl.copy()
    cloned.rho_raw[2] = raw_half.rho_raw[0]
    cloned = cloned.concat(raw_half)
    after = O.render(cloned, cfg, 0.7).image
    assert np.abs(after - before).max() < 1e-6


# ----------------------------------------------------------- adaptive control (test_trainer.cpp:150-231)
def _stats(m):
    return O.Stats.zeros(m)


def _adam(m):
    return {k: np.zeros(n) for k, n in zip(O.ADAM_KEYS, (m, m, 3 * m, 3 * m, 3 * m, 3 * m, 4 * m, 4 * m))}


def test_adaptive_control_prune_only():
    rng = O.Rng(223)
    c = O.random_cloud(rng, 5, 0.3, 0.05, 0.15)
    faint = O.kernels_to_cloud(c.s_min, [1e-4], [[0.5, 0.5, 0.5]], [[0.1, 0.1, 0.1]], [[1, 0, 0, 0]])
    c = c.concat(faint)
    nc, _, cnt = O.adaptive_control(rng, c, _adam(6), _stats(6))
    assert cnt == (1, 0, 0) and nc.m == 5


def test_adaptive_control_clone_and_split():
    c = O.kernels_to_cloud(2e-4, [0.8], [[0.1, 0.2, 0.3]], [[0.01, 0.01, 0.01]], [[1, 0, 0, 0]])
    st = _stats(1)
    st.grad2d_norm_accum[0], st.grad_count[0], st.grad3d_accum[0] = 1.0, 1, 1.0
    nc, na, cnt = O.adaptive_control(O.Rng(223), c, _adam(1), st)
    assert cnt == (0, 1, 0) and nc.m == 2
    np.testing.assert_allclose(nc.rho(), [0.4, 0.4], rtol=1e-9)
    assert np.linalg.norm(nc.pos[:3] - nc.pos[3:]) > 0.0
    assert na["m_rho"][1] == 0.0
    c = O.kernels_to_cloud(2e-4, [0.8], [[0.1, 0.2, 0.3]], [[0.1, 0.1, 0.1]], [[1, 0, 0, 0]])
    st = _stats(1)
    st.grad2d_norm_accum[0], st.grad_count[0] = 1.0, 1
    nc, _, cnt = O.adaptive_control(O.Rng(223), c, _adam(1), st)
    assert cnt == (0, 0, 1) and nc.m == 2
    np.testing.assert_allclose(nc.rho(), [0.4, 0.4], rtol=1e-9)
    np.testing.assert_allclose(nc.scale()[:, 0], [0.1 / 1.6] * 2, rtol=1e-9)
