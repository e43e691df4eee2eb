"""GPU train iteration (BASELINE configs[1]: render fwd/bwd + L1/D-SSIM + voxel
TV + Adam, trainer.cpp:268-319) against the same iteration composed from the
FP64 oracle, on identical views and TV sub-grid origins."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import oracle as O  # noqa: E402
from tests._helpers import rel_l2  # noqa: E402


def _oracle_step(oc, mom, t, theta, meas, inv_norm, origin, spacing, d, cfg, scanner):
    r = O.render(oc, scanner, theta)
    img = r.image * inv_norm
    l1, g1 = O.l1_loss(img, meas)
    ds, g2 = O.dssim_loss(img, meas)
    dL = (g1 + cfg.lambda_ssim * g2) * inv_norm
    g = O.Grads.zeros(oc.m)
    O.render_backward(oc, scanner, theta, r, dL, g, O.RasterOptions(), O.Stats.zeros(oc.m))
    grid = O.GridSpec((d, d, d), origin, spacing)
    vol = O.voxelize(oc, grid)
    tv, gtv = O.tv3d_loss(vol)
    O.voxelize_backward(oc, grid, gtv * cfg.lambda_tv, g)
    lrs = [O.lr_at(lr, cfg.lr_final_ratio, t, cfg.iters) for lr in
           (cfg.lr_position, cfg.lr_density, cfg.lr_scale, cfg.lr_rotation)]
    for name, lr in zip(("pos", "rho_raw", "scale_raw", "rot"), lrs):
        O.adam_step(getattr(oc, name), mom["m_" + name], mom["v_" + name], getattr(g, name), lr, t)
    O.normalize_rotations(oc)
    return l1, ds, tv


def test_train_steps_match_oracle():
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    import paper_2405_20693_b200 as P
    from paper_2405_20693_b200.train import TrainConfig, Trainer, random_subvolume_origin

    res, n_views = 64, 6
    scanner_o = O.test_scanner(res)
    angles = O.full_circle_angles(n_views)
    target = O.random_cloud(O.Rng(5), 80, 0.6, 0.05, 0.15)
    meas = np.stack([O.render(target, scanner_o, th).image for th in angles]).astype(np.float32)
    oc = O.random_cloud(O.Rng(6), 150, 0.6, 0.04, 0.12)
    f32 = [np.asarray(a, dtype=np.float32) for a in (oc.rho_raw, oc.pos, oc.scale_raw, oc.rot)]
    oc = O.Cloud.from_arrays(oc.s_min, *[a.astype(np.float64) for a in f32])
    p0 = {k: getattr(oc, k).copy() for k in ("rho_raw", "pos", "scale_raw", "rot")}
    ec = P.GaussianCloud(oc.s_min, *f32)
    cfg = TrainConfig(iters=100, output_dims=(32, 32, 32), tv_grid_dim=8, check_every=1)
    eng = P.Engine(0)
    tr = Trainer(eng, ec, P.ScannerConfig(detector_res_px=(res, res)), angles, torch.from_numpy(meas), cfg)
    inv_norm = 1.0 / float(meas.max())
    meas_norm = meas.astype(np.float64) * inv_norm
    mom = {f"{a}_{k}": np.zeros_like(getattr(oc, k)) for a in ("m", "v") for k in ("rho_raw", "pos", "scale_raw",
                                                                                      "rot")}
    spacing = tuple(2.0 / 32 for _ in range(3))
    rng = np.random.default_rng(0)
    for t, view in enumerate([2, 5, 0, 3], start=1):
        origin = random_subvolume_origin((-1,) * 3, (1,) * 3, spacing, 8, rng.random(3))
        out = tr.step(view=view, sub_origin=origin)
        l1, ds, tv = _oracle_step(oc, mom, t, angles[view], meas_norm[view], inv_norm, origin, spacing, 8, cfg,
                                  scanner_o)
        assert float(out["l1"]) == pytest.approx(l1, rel=1e-4)
        assert float(out["dssim"]) == pytest.approx(ds, rel=1e-3, abs=1e-6)
        assert float(out["tv"]) == pytest.approx(tv, rel=1e-3, abs=1e-7)
    for k in ("rho_raw", "pos", "scale_raw", "rot"):
        upd_gpu = getattr(ec, k).cpu().numpy().astype(np.float64) - p0[k]
        upd_ref = getattr(oc, k) - p0[k]
        assert rel_l2(upd_gpu, upd_ref) < 2e-2, k
    assert ec.grad_count.sum().item() > 0  # adaptive statistics accumulated (trainer.cpp:288)


def test_train_with_adaptive_control():
    """Iterations with densification inside the loop (trainer.cpp:321-323): the device
    adaptive-control pass applied to the trainer's own accumulated statistics matches the
    oracle on the same state, and training continues on the resized cloud."""
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    import paper_2405_20693_b200 as P
    from paper_2405_20693_b200.train import TrainConfig, Trainer

    res, n_views = 64, 6
    scanner_o = O.test_scanner(res)
    angles = O.full_circle_angles(n_views)
    target = O.random_cloud(O.Rng(5), 80, 0.6, 0.05, 0.15)
    meas = np.stack([O.render(target, scanner_o, th).image for th in angles]).astype(np.float32)
    oc = O.random_cloud(O.Rng(7), 300, 0.6, 0.01, 0.12)
    f32 = [np.asarray(a, dtype=np.float32) for a in (oc.rho_raw, oc.pos, oc.scale_raw, oc.rot)]
    cfg = TrainConfig(iters=100, output_dims=(32, 32, 32), tv_grid_dim=8, adaptive_start=2, densify_interval=3,
                      densify_grad_threshold=1e-6, prune_density_threshold=0.05)
    eng = P.Engine(0)
    tr = Trainer(eng, P.GaussianCloud(oc.s_min, *f32), P.ScannerConfig(detector_res_px=(res, res)), angles,
                 torch.from_numpy(meas), cfg)
    sizes = []
    for _ in range(4):  # t = 1..4; t = 5 is the first densification step
        sizes.append(tr.step()["kernels"])
    # state before the densification pass, as the oracle sees it
    c = tr.cloud
    h = lambda t: t.detach().cpu().numpy().astype(np.float64)
    ocl = O.Cloud(c.s_min, h(c.rho_raw), h(c.pos), h(c.scale_raw), h(c.rot))
    st = O.Stats(h(c.grad2d_norm_accum), c.grad_count.cpu().numpy().copy(), h(c.grad3d_accum))
    onc, oad, ocnt = O.adaptive_control(O.Rng(17), ocl, {k: h(v) for k, v in c.adam.items()}, st,
                                        cfg.prune_density_threshold, cfg.densify_grad_threshold,
                                        cfg.split_scale_threshold_frac, cfg.split_factor, (2.0, 2.0, 2.0))
    draws = torch.from_numpy(O.normal_draws(O.Rng(17), 6 * ocnt[2]))
    counts = tr.adaptive_control(gauss=draws)
    assert counts == tuple(ocnt) and sum(counts) > 0
    assert tr.cloud.size() == onc.m
    np.testing.assert_allclose(h(tr.cloud.pos), onc.pos, atol=2e-6, rtol=0)
    for k in O.ADAM_KEYS:
        np.testing.assert_array_equal(tr.cloud.adam[k].cpu().numpy(), oad[k].astype(np.float32))
    for _ in range(6):  # keeps training (and densifying at t = 5, 8) on the resized cloud
        out = tr.step()
        assert np.isfinite(float(out["total"]))
        sizes.append(out["kernels"])
    assert tr.grads.flat().numel() == 11 * tr.cloud.size()
    assert len(set(sizes)) > 1, sizes


@pytest.mark.parametrize("sync_free", [False, True])
def test_native_step_equals_python_step(sync_free):
    """sct_train_step (TrainConfig.native, one C-ABI call per iteration) issues the
    same launches in the same order as the call-by-call Python iteration: with the
    same seed, views, sub-grids and adaptive control, every loss value and every
    parameter / Adam moment / statistic is bitwise equal (deterministic reduction)."""
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    import paper_2405_20693_b200 as P
    from paper_2405_20693_b200.train import TrainConfig, Trainer

    res, n_views = 64, 6
    scanner_o = O.test_scanner(res)
    angles = O.full_circle_angles(n_views)
    target = O.random_cloud(O.Rng(5), 80, 0.6, 0.05, 0.15)
    meas = torch.from_numpy(np.stack([O.render(target, scanner_o, th).image for th in angles]).astype(np.float32))
    oc = O.random_cloud(O.Rng(7), 300, 0.6, 0.01, 0.12)
    f32 = [np.asarray(a, dtype=np.float32) for a in (oc.rho_raw, oc.pos, oc.scale_raw, oc.rot)]
    runs = []
    for native in (False, True):
        cfg = TrainConfig(iters=40, output_dims=(32, 32, 32), tv_grid_dim=8, adaptive_start=3, densify_interval=4,
                          densify_grad_threshold=1e-6, prune_density_threshold=0.05, seed=11, native=native,
                          sync_free=sync_free, check_every=5)
        eng = P.Engine(0)
        tr = Trainer(eng, P.GaussianCloud(oc.s_min, *f32), P.ScannerConfig(detector_res_px=(res, res)), angles,
                     meas, cfg)
        losses = [float(tr.step()["total"]) for _ in range(12)]
        c = tr.cloud
        state = [c.rho_raw, c.pos, c.scale_raw, c.rot, c.grad2d_norm_accum, c.grad_count, c.grad3d_accum,
                 *c.adam.values()]
        runs.append((losses, [x.detach().cpu().clone() for x in state]))
    (l0, s0), (l1, s1) = runs
    assert l0 == l1
    assert len(s0) == len(s1)
    for a, b in zip(s0, s1):
        assert torch.equal(a, b)


@pytest.mark.parametrize("sync_free", [False, True])
def test_native_trainer_equals_trainer(sync_free):
    """The engine-side train() loop (sct_trainer_*, csrc/trainer.cu) against the Python
    Trainer on the same seed: the same views, losses, adaptive-control counts and final
    cloud / Adam moments / statistics, bitwise (every draw from one std::mt19937_64)."""
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    import paper_2405_20693_b200 as P
    from paper_2405_20693_b200.train import NativeTrainer, TrainConfig, Trainer

    res, n_views = 64, 6
    scanner_o = O.test_scanner(res)
    angles = O.full_circle_angles(n_views)
    target = O.random_cloud(O.Rng(5), 80, 0.6, 0.05, 0.15)
    meas = torch.from_numpy(np.stack([O.render(target, scanner_o, th).image for th in angles]).astype(np.float32))
    oc = O.random_cloud(O.Rng(7), 300, 0.6, 0.01, 0.12)
    f32 = [np.asarray(a, dtype=np.float32) for a in (oc.rho_raw, oc.pos, oc.scale_raw, oc.rot)]
    cfg = TrainConfig(iters=40, output_dims=(32, 32, 32), tv_grid_dim=8, adaptive_start=3, densify_interval=4,
                      densify_grad_threshold=1e-6, prune_density_threshold=0.05, seed=13, sync_free=sync_free,
                      check_every=1)
    sc = P.ScannerConfig(detector_res_px=(res, res))
    tr = Trainer(P.Engine(0), P.GaussianCloud(oc.s_min, *f32), sc, angles, meas, cfg)
    py = []
    for _ in range(12):
        out = tr.step()
        py.append((out["view"], float(out["l1"]), float(out["dssim"]), float(out["tv"]), float(out["total"]),
                   out["kernels"]))
    nt = NativeTrainer(P.Engine(0), P.GaussianCloud(oc.s_min, *f32), sc, angles, meas, cfg)
    nat = []
    for _ in range(12):
        nt.step()
        r = nt.record()
        nat.append((r["view"], r["l1"], r["dssim"], r["tv"], r["total"], r["kernels"]))
    assert py == nat
    st = nt.state()
    c = tr.cloud
    for k in ("rho_raw", "pos", "scale_raw", "rot", "grad2d_norm_accum", "grad_count", "grad3d_accum"):
        np.testing.assert_array_equal(st[k], getattr(c, k).cpu().numpy(), err_msg=k)
    for k, v in c.adam.items():
        np.testing.assert_array_equal(st["adam"][k], v.cpu().numpy(), err_msg=k)
