"""Sync-free binning (Engine.set_capacity / sct_ctx_set_capacity): fixed-capacity
pair buffers instead of a host readback of each binning's pair count.

* tile and brick lists are identical to exact mode; images, volumes and
  gradients agree to FP32 rounding (the host-side work split of K3 / K4 / K8
  follows the pair count in exact mode and the capacity in capacity mode, which
  can regroup a list's 16-kernel chunks);
* a capacity below the pair count raises the overflow word (and only then),
  and the overflowing call is emptied rather than writing past its buffers;
* the train loop in sync-free mode reproduces exact mode (same densification
  events and kernel counts, parameters to FP32 rounding).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import oracle as O  # noqa: E402


def _need_cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")


def _cloud(P, seed=4, m=3000):
    oc = O.random_cloud(O.Rng(seed), m, 0.8, 0.005, 0.15)
    return P.GaussianCloud(oc.s_min, *[np.asarray(a, np.float32) for a in (oc.rho_raw, oc.pos, oc.scale_raw,
                                                                            oc.rot)])


@pytest.mark.parametrize("deterministic", [True, False])
def test_capacity_mode_matches_exact_mode(deterministic):
    """(atomic mode: the sync-free raster binning skips the per-item offset
    scan, which a later deterministic backward of the same state runs)"""
    _need_cuda()
    import paper_2405_20693_b200 as P
    c = _cloud(P)
    sc = P.ScannerConfig(detector_res_px=(200, 136))
    th = [0.2, 1.9, 4.0]
    up = torch.rand((3, 136, 200), device="cuda") - 0.5
    grid = P.grid_for_extent((-1, -1, -1), (1, 1, 1), (48, 40, 32))
    vup = torch.rand(grid.shape_zyx, device="cuda") - 0.5
    out = {}
    for mode in ("exact", "capacity"):
        eng = P.Engine(0, deterministic=deterministic)
        if mode == "capacity":
            eng.set_capacity(400000, 400000)
        f = eng.render(c, sc, th)
        g = P.CloudGrads(c.size())
        eng.render_backward(c, f, up, g)
        vol = eng.voxelize(c, grid)
        gv = P.CloudGrads(c.size())
        eng.voxelize_backward(c, grid, vup, gv)
        torch.cuda.synchronize()
        out[mode] = ([f.tile_lists(v) for v in range(3)], f.images.clone(), g.flat().clone(), vol.clone(),
                     gv.flat().clone(), f.n_pairs(), eng.take_overflow())
        f.free()
    a, b = out["exact"], out["capacity"]
    for (oa, ia), (ob, ib) in zip(a[0], b[0]):
        np.testing.assert_array_equal(oa, ob)
        np.testing.assert_array_equal(ia, ib)
    for name, x, y in zip(("images", "raster grads", "volume", "voxel grads"), a[1:5], b[1:5]):
        err = float(torch.linalg.norm((x - y).double()) / torch.linalg.norm(x.double()))
        assert err < 1e-5, (name, err)
    assert a[5] == b[5] and not b[6]


@pytest.mark.parametrize("deterministic", [True, False])
def test_capacity_overflow_is_flagged(deterministic):
    _need_cuda()
    import paper_2405_20693_b200 as P
    c = _cloud(P)
    eng = P.Engine(0, deterministic=deterministic)
    eng.set_capacity(1000, 1000)
    f = eng.render(c, P.ScannerConfig(detector_res_px=(128, 128)), [0.3])
    # an overflowing call is emptied (no pair is written beyond the buffers) and flagged
    assert f.n_pairs() == 0 and float(f.images.abs().sum()) == 0.0
    assert eng.take_overflow()
    assert not eng.take_overflow()  # cleared
    eng.voxelize(c, P.grid_for_extent((-1, -1, -1), (1, 1, 1), (32, 32, 32)))
    assert eng.take_overflow()
    f.free()


def test_sync_free_training_matches_exact_training():
    _need_cuda()
    import paper_2405_20693_b200 as P
    from paper_2405_20693_b200.train import TrainConfig, Trainer
    res, n_views = 48, 5
    scanner_o = O.test_scanner(res)
    angles = O.full_circle_angles(n_views)
    target = O.random_cloud(O.Rng(211), 40, 0.5, 0.06, 0.2)
    meas = torch.from_numpy(np.stack([O.render(target, scanner_o, th).image for th in angles]).astype(np.float32))
    init = O.random_cloud(O.Rng(212), 150, 0.6, 0.01, 0.12)
    f32 = [np.asarray(a, np.float32) for a in (init.rho_raw, init.pos, init.scale_raw, init.rot)]
    runs = {}
    for sync_free in (False, True):
        cfg = TrainConfig(iters=20, tv_grid_dim=8, output_dims=(32, 32, 32), adaptive_start=3, adaptive_end=18,
                          densify_interval=4, densify_grad_threshold=2e-5, prune_density_threshold=0.02, seed=5,
                          sync_free=sync_free, check_every=5)
        tr = Trainer(P.Engine(0, deterministic=True), P.GaussianCloud(init.s_min, *f32),
                     P.ScannerConfig(detector_res_px=(res, res)), angles, meas, cfg)
        sizes = [tr.step()["kernels"] for _ in range(cfg.iters)]
        torch.cuda.synchronize()
        runs[sync_free] = (sizes, tr.cloud)
    assert runs[False][0] == runs[True][0] and len(set(runs[True][0])) > 1
    for k in ("rho_raw", "pos", "scale_raw", "rot"):
        x, y = getattr(runs[False][1], k).double(), getattr(runs[True][1], k).double()
        assert float(torch.linalg.norm(x - y) / torch.linalg.norm(x)) < 1e-4, k


def test_atomic_forward_then_deterministic_backward():
    """A state binned in the atomic mode without per-item offsets gets them
    when the context switches to the deterministic backward."""
    _need_cuda()
    import paper_2405_20693_b200 as P
    c = _cloud(P)
    sc = P.ScannerConfig(detector_res_px=(160, 120))
    th = [0.5, 2.5]
    up = torch.rand((2, 120, 160), device="cuda") - 0.5
    ref = P.Engine(0, deterministic=True)
    ref.set_capacity(400000, 400000)
    f0 = ref.render(c, sc, th)
    g0 = P.CloudGrads(c.size())
    ref.render_backward(c, f0, up, g0)
    eng = P.Engine(0, deterministic=False)
    eng.set_capacity(400000, 400000)
    f = eng.render(c, sc, th)
    eng.set_deterministic(True)
    g = P.CloudGrads(c.size())
    eng.render_backward(c, f, up, g)
    torch.cuda.synchronize()
    assert torch.equal(g.flat(), g0.flat())  # same slots, same fixed-order sums
    assert not eng.take_overflow()
