"""Generate the committed golden fixtures (SURVEY.md §8c "Golden vectors").

The reference ships no golden vectors, so these are OUTPUTS OF THE REFERENCE
ITSELF: its unmodified sources (/root/reference/proj/core/src) compiled into
oracle/_ref/libsplatct_ref.so by `make -C oracle ref` (oracle/ref_capi.cpp over
the Eigen / nlohmann::json / libpng build shims in oracle/ref_shim/), called
through the same orc_* ABI as the FP64 restatement (oracle.using("reference")).
The containers are written by the reference's own io.cpp writers
(save_cloud / write_image / write_volume). tests/test_golden_cpu.py checks the
FP64 restatement (oracle/splatct_oracle.cpp) against them, and
tests/test_gpu_golden.py runs the engine against them.

Containers follow the reference formats (io.cpp): the cloud is a `.ckpt`
(io.cpp:171-182), images `.img` (:106-117), volumes `.vol` (:72-83), all fp32
little-endian behind a one-line JSON header; the integer binning (tile lists
per view, voxel brick lists) and the fp64 gradients are `.npz`.

Run from the repo root (needs /root/reference or a prebuilt oracle/_ref):
    python tests/golden/make_golden.py
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402

# Raster case: 400 anisotropic, rotated kernels (tests/helpers.hpp:30-48 stream),
# a 100x72 detector (partial edge tiles: 100 = 6*16 + 4), three views, and two
# option sets (rectified default; biased with frozen Jacobian and no low-pass).
RASTER = dict(seed=41, m=400, pos_radius=0.6, scale_min=0.03, scale_max=0.15, res=(100, 72),
              thetas=[0.37, 2.1, 4.4], upstream_seed=2)
OPTION_SETS = {
    "rectified": dict(mode=0),
    "biased_frozen_nolp": dict(mode=1, lowpass_eps_px=0.0, freeze_jacobian=True),
}
# Narrow-kernel case (rasterizer.cpp:44-50,151 with lowpass_eps_px = 0 / 0.1,
# test_rasterizer.cpp:49,186): sub-pixel kernels, projected sigma 0.03-0.3 px,
# where exp(-1/2 d^T Q d) falls by orders of magnitude between neighbouring pixels.
NARROW = dict(seed=43, m=400, pos_radius=0.6, scale_min=0.0008, scale_max=0.012)
NARROW_SETS = {
    "narrow_eps0": dict(mode=0, lowpass_eps_px=0.0),
    "narrow_eps01": dict(mode=0, lowpass_eps_px=0.1),
}
# Voxel case: non-cubic grid with dims not multiples of 8 and an off-centre origin.
VOXEL = dict(lo=(-1.0, -0.9, -0.8), hi=(1.0, 0.9, 0.7), dims=(21, 18, 13), upstream_seed=3)


def f32_cloud(c):
    return O.Cloud.from_arrays(c.s_min, *[np.asarray(a, np.float32).astype(np.float64)
                                          for a in (c.rho_raw, c.pos, c.scale_raw, c.rot)])


def raster_case(cloud, opt_name):
    cfg = O.ScannerConfig(detector_res_px=RASTER["res"])
    opts = O.RasterOptions(**{**OPTION_SETS, **NARROW_SETS}[opt_name])
    w, h = RASTER["res"]
    rng = O.Rng(RASTER["upstream_seed"])
    images, ups, offs, idxs = [], [], [], []
    grads = O.Grads.zeros(cloud.m)
    stats = O.Stats.zeros(cloud.m)
    for th in RASTER["thetas"]:
        r = O.render(cloud, cfg, th, opts)
        dL = O.random_image(rng, w, h, -1.0, 1.0).astype(np.float32).astype(np.float64)
        O.render_backward(cloud, cfg, th, r, dL, grads, opts, stats)
        off, idx = r.tile_lists()
        images.append(r.image)
        ups.append(dL)
        offs.append(off)
        idxs.append(idx)
    return dict(images=np.stack(images), upstream=np.stack(ups), offsets=offs, idx=idxs, grads=grads, stats=stats)


def voxel_case(cloud):
    grid = O.grid_for_extent(VOXEL["lo"], VOXEL["hi"], VOXEL["dims"])
    vol = O.voxelize(cloud, grid)
    rng = O.Rng(VOXEL["upstream_seed"])
    n = int(np.prod(grid.dims))
    dL = O.random_image(rng, n, 1, -1.0, 1.0).astype(np.float32).astype(np.float64).reshape(grid.shape_zyx)
    g = O.Grads.zeros(cloud.m)
    O.voxelize_backward(cloud, grid, dL, g)
    off, idx = O.voxel_bins(cloud, grid)
    return dict(grid=grid, volume=vol, upstream=dL, grads=g, offsets=off, idx=idx)


def main():
    with O.using("reference"):
        _main()


def _main():
    rio = O.reference_io()

    c = f32_cloud(O.random_cloud(O.Rng(RASTER["seed"]), RASTER["m"], RASTER["pos_radius"], RASTER["scale_min"],
                                 RASTER["scale_max"]))
    rio.save_cloud(c, os.path.join(HERE, "cloud.ckpt"))
    cn = f32_cloud(O.random_cloud(O.Rng(NARROW["seed"]), NARROW["m"], NARROW["pos_radius"], NARROW["scale_min"],
                                  NARROW["scale_max"]))
    rio.save_cloud(cn, os.path.join(HERE, "cloud_narrow.ckpt"))
    manifest = {"generator": "tests/golden/make_golden.py (the reference's own sources, oracle/_ref)",
                "raster": RASTER, "option_sets": {**OPTION_SETS, **NARROW_SETS}, "narrow": NARROW,
                "narrow_sets": list(NARROW_SETS), "voxel": VOXEL, "cases": {}}
    for name in list(OPTION_SETS) + list(NARROW_SETS):
        r = raster_case(cn if name in NARROW_SETS else c, name)
        for v in range(len(RASTER["thetas"])):
            rio.write_image(r["images"][v], os.path.join(HERE, f"raster_{name}_view{v}.img"))
        rio.write_image(r["upstream"].reshape(-1, RASTER["res"][0]), os.path.join(HERE, f"raster_{name}_dL.img"))
        g, st = r["grads"], r["stats"]
        np.savez_compressed(
            os.path.join(HERE, f"raster_{name}.npz"),
            **{f"offsets{v}": r["offsets"][v] for v in range(len(RASTER["thetas"]))},
            **{f"idx{v}": r["idx"][v] for v in range(len(RASTER["thetas"]))},
            g_rho_raw=g.rho_raw, g_pos=g.pos, g_scale_raw=g.scale_raw, g_rot=g.rot,
            grad2d_norm_accum=st.grad2d_norm_accum, grad_count=st.grad_count, grad3d_accum=st.grad3d_accum)
        manifest["cases"][name] = {"pairs_per_view": [int(len(i)) for i in r["idx"]]}
    vx = voxel_case(c)
    gr = vx["grid"]
    rio.write_volume(vx["volume"], gr, os.path.join(HERE, "voxel_volume.vol"))
    rio.write_volume(vx["upstream"], gr, os.path.join(HERE, "voxel_dL.vol"))
    g = vx["grads"]
    np.savez_compressed(os.path.join(HERE, "voxel.npz"), offsets=vx["offsets"], idx=vx["idx"],
                        g_rho_raw=g.rho_raw, g_pos=g.pos, g_scale_raw=g.scale_raw, g_rot=g.rot)
    manifest["cases"]["voxel"] = {"pairs": int(len(vx["idx"]))}
    with open(os.path.join(HERE, "manifest.json"), "w") as f:
        json.dump(manifest, f, indent=1)
    print(json.dumps(manifest["cases"]))


if __name__ == "__main__":
    main()
