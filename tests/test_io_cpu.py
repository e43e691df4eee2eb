"""Container I/O (io.cpp:20-213), re-expressing tests/test_io.cpp and the
checkpoint round trip of tests/test_gaussian_cloud.cpp:167-188. CPU only."""
import json

import numpy as np
import pytest
import torch

import paper_2405_20693_b200 as P
from paper_2405_20693_b200 import io as sio
from paper_2405_20693_b200 import scenes


def _cloud(m=7, seed=29):
    ca = scenes.random_cloud(m, seed=seed)
    return P.GaussianCloud(ca.s_min, ca.rho_raw, ca.pos, ca.scale_raw, ca.rot, device="cpu")


def test_cloud_round_trip_and_byte_identical_rewrite(tmp_path):
    c = _cloud()
    p = str(tmp_path / "c.ckpt")
    sio.save_cloud(c, p)
    b = sio.load_cloud(p, device="cpu")
    assert b.size() == c.size() and b.s_min == pytest.approx(c.s_min)
    for k in ("rho_raw", "pos", "scale_raw", "rot"):
        assert torch.equal(getattr(b, k), getattr(c, k))
    sio.save_cloud(b, p + "2")
    sio.save_cloud(sio.load_cloud(p + "2", device="cpu"), p + "3")
    assert open(p + "2", "rb").read() == open(p + "3", "rb").read()
    # header as the reference writes it (io.cpp:171-182), payload fp32 LE in field order
    raw = open(p, "rb").read()
    line, payload = raw.split(b"\n", 1)
    h = json.loads(line)
    assert h["kind"] == "gaussian_cloud" and h["count"] == 7
    assert h["fields"] == ["rho_raw", "positions_mm", "scales_raw", "rotations_wxyz"]
    assert len(payload) == 4 * 11 * 7
    np.testing.assert_array_equal(np.frombuffer(payload[:28], "<f4"), c.rho_raw.numpy())


def test_cloud_adam_extension(tmp_path):
    c = _cloud()
    for k, t in c.adam.items():
        t.copy_(torch.arange(t.numel(), dtype=torch.float32) + len(k))
    p = str(tmp_path / "a.ckpt")
    sio.save_cloud(c, p, include_adam=True)
    b = sio.load_cloud(p, device="cpu")
    for k in c.adam:
        assert torch.equal(b.adam[k], c.adam[k])
    # without the extension the moments load as zeros (io.cpp:201-211)
    sio.save_cloud(c, p + "0")
    assert all(not t.any() for t in sio.load_cloud(p + "0", device="cpu").adam.values())


def test_volume_and_image_round_trip(tmp_path):
    rng = np.random.default_rng(301)
    grid = P.grid_for_extent((-1, -1, -1), (1, 1, 1), (9, 7, 5))
    v = rng.uniform(-2, 2, grid.shape_zyx).astype(np.float32)
    p = str(tmp_path / "v.vol")
    sio.write_volume(v, grid, p)
    back, g2 = sio.read_volume(p)
    np.testing.assert_array_equal(back, v)
    assert g2.dims == grid.dims and np.allclose(g2.origin_mm, grid.origin_mm)
    sio.write_volume(back, g2, p + "2")
    b2, g3 = sio.read_volume(p + "2")
    sio.write_volume(b2, g3, p + "3")
    assert open(p + "2", "rb").read() == open(p + "3", "rb").read()
    img = rng.uniform(-1, 3, (8, 12)).astype(np.float32)
    sio.write_image(img, str(tmp_path / "i.img"), {"theta_rad": 1.25})
    bi, meta = sio.read_image(str(tmp_path / "i.img"))
    np.testing.assert_array_equal(bi, img)
    assert meta["theta_rad"] == pytest.approx(1.25)


def test_format_errors(tmp_path):  # test_io.cpp:56-100
    p = str(tmp_path / "bad.bin")
    with pytest.raises(P.DataError):
        sio.read_volume(str(tmp_path / "missing.vol"))
    sio.write_image(np.zeros((4, 4), np.float32), p)
    with pytest.raises(sio.FileFormatError):
        sio.read_volume(p)
    with open(p, "wb") as f:
        f.write(b'{"kind":"volume","dims":[8,8,8],"spacing_mm":[1,1,1],"origin_mm":[0,0,0],"dtype":"float32",'
                b'"endianness":"little"}\n')
        f.write(np.arange(4, dtype="<f4").tobytes())
    with pytest.raises(sio.FileFormatError):
        sio.read_volume(p)
    with open(p, "wb") as f:
        f.write(b"not json at all\n")
    with pytest.raises(sio.FileFormatError):
        sio.read_volume(p)
    with open(p, "wb") as f:
        f.write(b'{"kind":"volume","dims":[2,2,2],"spacing_mm":[1,1,1],"origin_mm":[0,0,0],"dtype":"float64",'
                b'"endianness":"little"}\n')
    with pytest.raises(sio.FileFormatError):
        sio.read_volume(p)
