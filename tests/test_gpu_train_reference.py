"""The engine's training loop against THE REFERENCE'S OWN `train`
(trainer.cpp:232-345, compiled unmodified into oracle/_ref), on the same seed.

The engine draws from the reference's single std::mt19937_64 stream
(engine.HostRng: std::shuffle of the view order, the TV sub-volume origin, the
adaptive-control split draws, in the reference's order), so both loops pick
the same views, the same sub-grids and the same densification events:

* the kernel count after every iteration is identical (prune / clone / split
  decisions, densification at the same iterations);
* per-iteration L1, D-SSIM and TV values agree to the fp32 bar;
* the parameter updates agree to 2e-2 relative L2 after the whole run
  (fp32 Adam against fp64 Adam: sign-like updates of near-zero gradients
  differ, as in test_gpu_train.py).

Plus the reference's bit-reproducibility test (test_trainer.cpp:87-105) on the
device: two seeded runs give bit-identical clouds (deterministic reduction).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import oracle as O  # noqa: E402
from tests._helpers import rel_l2  # noqa: E402


def _scene(res=48, n_views=5, m=120):
    scanner = O.test_scanner(res)
    angles = O.full_circle_angles(n_views)
    target = O.random_cloud(O.Rng(211), 40, 0.5, 0.06, 0.2)
    meas = np.stack([O.render(target, scanner, th).image for th in angles]).astype(np.float32)
    init = O.random_cloud(O.Rng(212), m, 0.6, 0.01, 0.12)
    f32 = [np.asarray(a, dtype=np.float32) for a in (init.rho_raw, init.pos, init.scale_raw, init.rot)]
    init = O.Cloud.from_arrays(init.s_min, *[a.astype(np.float64) for a in f32])
    return scanner, angles, meas, init, f32


def _engine_run(P, scanner_res, angles, meas, f32, s_min, tc, deterministic=True):
    from paper_2405_20693_b200.train import TrainConfig, Trainer
    cfg = TrainConfig(iters=tc.iters, lr_position=tc.lr_position, lr_density=tc.lr_density, lr_scale=tc.lr_scale,
                      lr_rotation=tc.lr_rotation, lr_final_ratio=tc.lr_final_ratio, lambda_ssim=tc.lambda_ssim,
                      lambda_tv=tc.lambda_tv, tv_grid_dim=tc.tv_grid_dim, adaptive_start=tc.adaptive_start,
                      adaptive_end=tc.adaptive_end, densify_interval=tc.densify_interval,
                      densify_grad_threshold=tc.densify_grad_threshold,
                      prune_density_threshold=tc.prune_density_threshold,
                      split_scale_threshold_frac=tc.split_scale_threshold_frac, split_factor=tc.split_factor,
                      output_dims=tc.output_dims, seed=tc.seed, mode=tc.mode)
    eng = P.Engine(0, deterministic=deterministic)
    tr = Trainer(eng, P.GaussianCloud(s_min, *[a.copy() for a in f32]),
                 P.ScannerConfig(detector_res_px=(scanner_res, scanner_res)), angles, torch.from_numpy(meas), cfg)
    hist = []
    for _ in range(tc.iters):
        out = tr.step()
        hist.append((out["iter"], float(out["l1"]), float(out["dssim"]), float(out["tv"]), float(out["total"]),
                     out["kernels"], out["view"]))
    torch.cuda.synchronize()
    return tr, hist


def _cfg(**kw):
    tc = O.TrainConfig(iters=24, tv_grid_dim=8, output_dims=(32, 32, 32), adaptive_start=3, adaptive_end=21,
                       densify_interval=4, densify_grad_threshold=2e-5, prune_density_threshold=0.02,
                       history_interval=1, seed=5)
    for k, v in kw.items():
        setattr(tc, k, v)
    return tc


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref (the compiled reference) not built")
def test_train_loop_matches_reference_train():
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    import paper_2405_20693_b200 as P
    scanner, angles, meas, init, f32 = _scene()
    tc = _cfg()
    rc, radam, rstats, rhist = O.train_reference(init, scanner, angles, meas.astype(np.float64), tc)
    tr, ehist = _engine_run(P, scanner.detector_res_px[0], angles, meas, f32, init.s_min, tc)
    assert len(rhist) == tc.iters
    # same densification events, same kernel counts after every iteration
    r_kernels = [int(r[5]) for r in rhist]
    e_kernels = [h[5] for h in ehist]
    assert e_kernels == r_kernels, (e_kernels, r_kernels)
    assert len(set(r_kernels)) > 1, "the run must densify / prune"
    for r, e in zip(rhist, ehist):
        assert int(r[0]) == e[0]
        assert e[1] == pytest.approx(r[1], rel=2e-3), ("l1", e[0])
        assert e[2] == pytest.approx(r[2], rel=2e-3, abs=1e-6), ("dssim", e[0])
        assert e[3] == pytest.approx(r[3], rel=2e-3, abs=1e-7), ("tv", e[0])
    # parameter updates of the whole run
    got = {k: getattr(tr.cloud, k).cpu().numpy().astype(np.float64) for k in ("rho_raw", "pos", "scale_raw", "rot")}
    for k in ("rho_raw", "pos", "scale_raw", "rot"):
        assert got[k].shape == getattr(rc, k).shape, k
        assert rel_l2(got[k], getattr(rc, k)) < 2e-2, k
    # the statistics the reference carries at the end (accumulated since the last reset)
    np.testing.assert_array_equal(tr.cloud.grad_count.cpu().numpy(), rstats.grad_count)


def test_seeded_training_is_bit_reproducible():  # test_trainer.cpp:87-105
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    import paper_2405_20693_b200 as P
    scanner, angles, meas, init, f32 = _scene(res=32, n_views=4, m=3)
    tc = _cfg(iters=25, adaptive_start=0, adaptive_end=0, lambda_tv=0.05, seed=5)
    a, ha = _engine_run(P, 32, angles, meas, f32, init.s_min, tc)
    b, hb = _engine_run(P, 32, angles, meas, f32, init.s_min, tc)
    assert [h[6] for h in ha] == [h[6] for h in hb]  # same view sequence
    for k in ("rho_raw", "pos", "scale_raw", "rot"):
        assert torch.equal(getattr(a.cloud, k), getattr(b.cloud, k)), k
