"""Full-size parity numbers (cfg3 sampled views, cfg4 slab) -> profiles/r01_parity_fullsize.json.
Same comparisons as tests/test_gpu_fullsize.py, reporting the measured errors."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2405_20693_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2405_20693_b200 import scenes  # noqa: E402


def rel(a, b):
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


out = {"bars": {"lists": "bit-exact", "images/volumes": "rel L2 <= 1e-4", "gradients": "rel L2 <= 1e-3"}}
w, ca, thetas, vol = bench.make_workload()
f32 = [np.asarray(a, dtype=np.float32) for a in (ca.rho_raw, ca.pos, ca.scale_raw, ca.rot)]
ec = P.GaussianCloud(ca.s_min, *f32)
oc = O.Cloud.from_arrays(ca.s_min, *[a.astype(np.float64) for a in f32])
for det in (True, False):
    eng = P.Engine(0, deterministic=det)
    res = w.res
    views = [0, 37]
    up = np.random.default_rng(2).uniform(-1, 1, (len(views), res, res)).astype(np.float32)
    fwd = eng.render(ec, P.ScannerConfig(detector_res_px=(res, res)), [thetas[v] for v in views])
    g = P.CloudGrads(ec.size())
    eng.render_backward(ec, fwd, torch.from_numpy(up).cuda(), g)
    imgs = fwd.images.cpu().numpy()
    og = O.Grads.zeros(oc.m)
    rec = {"views": views, "pairs": [], "lists_equal": [], "image_rel_l2": []}
    for k, v in enumerate(views):
        r = O.render(oc, O.test_scanner(res), thetas[v])
        off_o, idx_o = r.tile_lists()
        off_e, idx_e = fwd.tile_lists(k)
        rec["pairs"].append(int(off_o[-1]))
        rec["lists_equal"].append(bool(np.array_equal(off_e, off_o) and np.array_equal(idx_e, idx_o)))
        rec["image_rel_l2"].append(rel(imgs[k], r.image))
        O.render_backward(oc, O.test_scanner(res), thetas[v], r, up[k].astype(np.float64), og)
    rec["grad_rel_l2"] = {n: rel(a.cpu().numpy(), b) for n, a, b in
                          zip(("rho_raw", "pos", "scale_raw", "rot"), g.tensors(),
                              (og.rho_raw, og.pos, og.scale_raw, og.rot))}
    out["cfg3_" + ("deterministic" if det else "atomic")] = rec
c4 = scenes.make_cloud(4, vol=vol)
f32 = [np.asarray(a, dtype=np.float32) for a in (c4.rho_raw, c4.pos, c4.scale_raw, c4.rot)]
ec4 = P.GaussianCloud(c4.s_min, *f32)
oc4 = O.Cloud.from_arrays(c4.s_min, *[a.astype(np.float64) for a in f32])
eng = P.Engine(0)
n = scenes.CONFIGS[4].n_vox
z0, nz = n // 2 - 8, 16
grid = P.grid_for_extent((-1, -1, -1), (1, 1, 1), (n, n, n))
og = O.GridSpec((n, n, nz), (grid.origin_mm[0], grid.origin_mm[1], grid.origin_mm[2] + z0 * grid.spacing_mm[2]),
                tuple(grid.spacing_mm))
eg = P.GridSpec((n, n, nz), og.origin_mm, og.spacing_mm)
vol_e = eng.voxelize(ec4, eg).cpu().numpy()
vol_o = O.voxelize(oc4, og)
upv = np.random.default_rng(3).uniform(-1, 1, og.shape_zyx)
ge = P.CloudGrads(ec4.size())
eng.voxelize_backward(ec4, eg, torch.from_numpy(upv.astype(np.float32)).cuda(), ge)
gov = O.Grads.zeros(oc4.m)
O.voxelize_backward(oc4, og, upv, gov)
off_e, idx_e = eng.voxel_bins(ec4, eg)
off_o, idx_o = O.voxel_bins(oc4, og)
out["cfg4_slab"] = {"grid": [n, n, nz], "z0": z0, "pairs": int(off_o[-1]),
                    "bricks_equal": bool(np.array_equal(off_e, off_o) and np.array_equal(idx_e, idx_o)),
                    "volume_rel_l2": rel(vol_e, vol_o),
                    "grad_rel_l2": {nm: rel(a.cpu().numpy(), b) for nm, a, b in
                                    zip(("rho_raw", "pos", "scale_raw", "rot"), ge.tensors(),
                                        (gov.rho_raw, gov.pos, gov.scale_raw, gov.rot))}}
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(out, open(os.path.join(ROOT, "gpurun_out", "parity_fullsize.json"), "w"), indent=1)
print(json.dumps(out, indent=1))
