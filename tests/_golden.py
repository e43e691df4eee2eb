"""Loader for the committed golden fixtures (tests/golden/, made by make_golden.py)."""
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def manifest():
    with open(os.path.join(GOLDEN, "manifest.json")) as f:
        return json.load(f)


RASTER_SETS = ["rectified", "biased_frozen_nolp", "narrow_eps0", "narrow_eps01"]


def cloud_arrays(case: str = "rectified"):
    """(s_min, rho_raw, pos, scale_raw, rot) fp32 from the case's cloud
    (cloud_narrow.ckpt for the narrow-kernel sets, else cloud.ckpt)."""
    from paper_2405_20693_b200 import io as sio
    narrow = case in manifest().get("narrow_sets", [])
    c = sio.load_cloud(os.path.join(GOLDEN, "cloud_narrow.ckpt" if narrow else "cloud.ckpt"), device="cpu")
    return (c.s_min,) + tuple(getattr(c, k).numpy() for k in ("rho_raw", "pos", "scale_raw", "rot"))


def raster(name):
    from paper_2405_20693_b200 import io as sio
    man = manifest()
    nv = len(man["raster"]["thetas"])
    imgs = np.stack([sio.read_image(os.path.join(GOLDEN, f"raster_{name}_view{v}.img"))[0] for v in range(nv)])
    w, h = man["raster"]["res"]
    dL = sio.read_image(os.path.join(GOLDEN, f"raster_{name}_dL.img"))[0].reshape(nv, h, w)
    z = dict(np.load(os.path.join(GOLDEN, f"raster_{name}.npz")))
    return man, imgs, dL, z


def voxel():
    from paper_2405_20693_b200 import io as sio
    vol, grid = sio.read_volume(os.path.join(GOLDEN, "voxel_volume.vol"))
    dL, _ = sio.read_volume(os.path.join(GOLDEN, "voxel_dL.vol"))
    z = dict(np.load(os.path.join(GOLDEN, "voxel.npz")))
    return grid, vol, dL, z
