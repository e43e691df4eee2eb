#!/usr/bin/env python
"""One pass of every engine kernel family inside cudaProfilerStart/Stop, for
`ncu --profile-from-start off` captures (tools/profile_round2.sh):
  * cfg3 render fwd + bwd (75 views at 512^2, 100k Gaussians; --reduction),
  * cfg4 voxelize + voxelize_backward (256^3, 200k Gaussians),
  * cfg2 train iterations (render 1 view, L1/D-SSIM, TV, Adam) and one
    adaptive-control pass.
Everything is warmed up first; the profiled pass repeats the same calls."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_20693_b200 as P  # noqa: E402
from paper_2405_20693_b200 import scenes  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reduction", default="atomic", choices=["atomic", "deterministic"])
    ap.add_argument("--parts", default="raster,voxel,train")
    a = ap.parse_args()
    parts = a.parts.split(",")
    eng = P.Engine(0, deterministic=a.reduction == "deterministic")
    work = []
    if "raster" in parts:
        w = scenes.CONFIGS[3]
        vol = scenes.phantom(w.n_vox)
        ca = scenes.make_cloud(3, vol=vol)
        cl = P.GaussianCloud(ca.s_min, ca.rho_raw, ca.pos, ca.scale_raw, ca.rot)
        sc = P.ScannerConfig(detector_res_px=(w.res, w.res))
        th = P.full_circle_angles(w.n_views)
        dl = torch.rand((w.n_views, w.res, w.res), device="cuda") * 2 - 1
        g = P.CloudGrads(cl.size())

        def raster():
            f = eng.render(cl, sc, th)
            eng.render_backward(cl, f, dl, g)
            f.free()
        work.append(raster)
    if "voxel" in parts:
        w4 = scenes.CONFIGS[4]
        ca4 = scenes.make_cloud(4)
        cl4 = P.GaussianCloud(ca4.s_min, ca4.rho_raw, ca4.pos, ca4.scale_raw, ca4.rot)
        grid = P.grid_for_extent((-1, -1, -1), (1, 1, 1), (w4.n_vox,) * 3)
        up = torch.rand(grid.shape_zyx, device="cuda") * 2 - 1
        g4 = P.CloudGrads(cl4.size())

        def voxel():
            _, vs = eng.voxelize(cl4, grid, keep_state=True)
            eng.voxelize_backward(cl4, grid, up, g4, state=vs)
            vs.free()
        work.append(voxel)
    if "train" in parts:
        from paper_2405_20693_b200.train import TrainConfig, Trainer
        w2 = scenes.CONFIGS[2]
        ca2 = scenes.make_cloud(2)
        angles = P.full_circle_angles(w2.n_views)
        sc2 = P.ScannerConfig(detector_res_px=(w2.res, w2.res))
        tgt = P.GaussianCloud(ca2.s_min, ca2.rho_raw * 1.1, ca2.pos, ca2.scale_raw, ca2.rot)
        f = eng.render(tgt, sc2, angles)
        meas = f.images.clone()
        f.free()
        cfg = TrainConfig(iters=1000, output_dims=(w2.n_vox,) * 3, tv_grid_dim=32, check_every=0,
                          densify_grad_threshold=2e-6)
        tr = Trainer(eng, P.GaussianCloud(ca2.s_min, ca2.rho_raw, ca2.pos, ca2.scale_raw, ca2.rot), sc2, angles,
                     meas, cfg)

        def train():
            tr.step()
            tr.step()
            tr.adaptive_control()
        work.append(train)
    for _ in range(3):
        for f in work:
            f()
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    for f in work:
        f()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print("profile_step: done", parts, file=sys.stderr)


if __name__ == "__main__":
    main()
