"""Checkpoint / container I/O on the device (io.cpp:20-213).

* the device fast path (one pinned staging buffer and one host-to-device copy
  on load, one device-to-host copy on save) round-trips a cloud with its Adam
  moments bit-exactly;
* files written from device memory are read by THE REFERENCE's own io.cpp
  (oracle/_ref) and reference-written files load onto the device unchanged;
* resume: training N iterations, checkpointing (parameters + the Adam-moment
  extension), reloading and training M more gives the same cloud, bit for bit,
  as N + M uninterrupted iterations (deterministic reduction).
"""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import oracle as O  # noqa: E402


def _need_cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")


def test_device_checkpoint_round_trip(tmp_path):
    _need_cuda()
    import paper_2405_20693_b200 as P
    from paper_2405_20693_b200 import io as sio
    from paper_2405_20693_b200 import scenes
    ca = scenes.random_cloud(5000, seed=3)
    c = P.GaussianCloud(ca.s_min, ca.rho_raw, ca.pos, ca.scale_raw, ca.rot)
    for k, t in c.adam.items():
        t.copy_(torch.randn(t.numel(), device="cuda"))
    p = str(tmp_path / "c.ckpt")
    sio.save_cloud(c, p, include_adam=True)
    b = sio.load_cloud(p)
    assert b.rho_raw.is_cuda and b.size() == c.size() and b.s_min == c.s_min
    for k in ("rho_raw", "pos", "scale_raw", "rot"):
        assert torch.equal(getattr(b, k), getattr(c, k)), k
    for k in c.adam:
        assert torch.equal(b.adam[k], c.adam[k]), k
    vol = torch.rand((13, 18, 21), device="cuda")
    g = P.GridSpec((21, 18, 13), (-1.0, -0.9, -0.8), (0.1, 0.1, 0.11))
    sio.write_volume(vol, g, str(tmp_path / "v.vol"))
    v2, g2 = sio.read_volume(str(tmp_path / "v.vol"))
    np.testing.assert_array_equal(v2, vol.cpu().numpy())
    assert tuple(g2.dims) == (21, 18, 13)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref (the compiled reference) not built")
def test_device_files_and_reference_io(tmp_path):
    _need_cuda()
    import paper_2405_20693_b200 as P
    from paper_2405_20693_b200 import io as sio
    rio = O.reference_io()
    oc = O.random_cloud(O.Rng(9), 777)
    f32 = [np.asarray(a, dtype=np.float32) for a in (oc.rho_raw, oc.pos, oc.scale_raw, oc.rot)]
    c = P.GaussianCloud(oc.s_min, *f32)
    sio.save_cloud(c, str(tmp_path / "dev.ckpt"), include_adam=True)  # the reference ignores the extension
    back = rio.load_cloud(str(tmp_path / "dev.ckpt"))
    for k, a in zip(("rho_raw", "pos", "scale_raw", "rot"), f32):
        np.testing.assert_array_equal(getattr(back, k), a.astype(np.float64))
    rio.save_cloud(back, str(tmp_path / "ref.ckpt"))
    d = sio.load_cloud(str(tmp_path / "ref.ckpt"))
    for k, a in zip(("rho_raw", "pos", "scale_raw", "rot"), f32):
        np.testing.assert_array_equal(getattr(d, k).cpu().numpy(), a)


def test_resume_from_checkpoint_is_bit_exact(tmp_path):
    _need_cuda()
    import paper_2405_20693_b200 as P
    from paper_2405_20693_b200 import io as sio
    from paper_2405_20693_b200.train import TrainConfig, Trainer
    res, n_views = 48, 5
    scanner_o = O.test_scanner(res)
    angles = O.full_circle_angles(n_views)
    target = O.random_cloud(O.Rng(5), 60, 0.6, 0.05, 0.15)
    meas = torch.from_numpy(np.stack([O.render(target, scanner_o, th).image for th in angles]).astype(np.float32))
    init = O.random_cloud(O.Rng(6), 200, 0.6, 0.02, 0.12)
    f32 = [np.asarray(a, dtype=np.float32) for a in (init.rho_raw, init.pos, init.scale_raw, init.rot)]
    cfg = TrainConfig(iters=40, output_dims=(32, 32, 32), tv_grid_dim=8, adaptive_start=40, adaptive_end=40)
    views = [3, 1, 4, 0, 2, 2, 0, 1, 3, 4, 1, 0]
    rng = np.random.default_rng(1)
    origins = [tuple(rng.uniform(-1.0, 0.7, 3)) for _ in views]
    sc = P.ScannerConfig(detector_res_px=(res, res))

    def trainer(cloud):
        return Trainer(P.Engine(0, deterministic=True), cloud, sc, angles, meas, cfg)

    full = trainer(P.GaussianCloud(init.s_min, *f32))
    for v, o in zip(views, origins):
        full.step(view=v, sub_origin=o)
    first = trainer(P.GaussianCloud(init.s_min, *f32))
    for v, o in zip(views[:7], origins[:7]):
        first.step(view=v, sub_origin=o)
    p = str(tmp_path / "resume.ckpt")
    sio.save_cloud(first.cloud, p, include_adam=True)
    second = trainer(sio.load_cloud(p))
    second.t = first.t  # iteration counter: Adam bias correction and the lr schedule (trainer.cpp:310-319)
    for v, o in zip(views[7:], origins[7:]):
        second.step(view=v, sub_origin=o)
    torch.cuda.synchronize()
    for k in ("rho_raw", "pos", "scale_raw", "rot"):
        assert torch.equal(getattr(second.cloud, k), getattr(full.cloud, k)), k
    for k in full.cloud.adam:
        assert torch.equal(second.cloud.adam[k], full.cloud.adam[k]), k
