#!/usr/bin/env python
"""Times render fwd+bwd (and voxelize fwd+bwd) on any BASELINE config on one
GPU, for robustness/scaling checks beyond bench.py's headline workload.
  python tools/bench_configs.py --config 5 [--views 100] [--steps 3]
Prints one JSON line per config."""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_20693_b200 as P  # noqa: E402
from paper_2405_20693_b200 import scenes  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, nargs="+", default=[1, 3, 5])
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--voxel", action="store_true")
    a = ap.parse_args()
    eng = P.Engine(0, deterministic=False)  # parallel-atomic backward, as bench.py
    for cfg in a.config:
        w = scenes.CONFIGS[cfg]
        t0 = time.time()
        vol = scenes.phantom(w.n_vox)
        ca = scenes.make_cloud(cfg, vol=vol)
        gen = time.time() - t0
        cloud = P.GaussianCloud(ca.s_min, ca.rho_raw, ca.pos, ca.scale_raw, ca.rot)
        out = {"config": cfg, "workload": w.description, "fixture_s": round(gen, 1)}
        if w.n_views:
            thetas = P.full_circle_angles(w.n_views)
            sc = P.ScannerConfig(detector_res_px=(w.res, w.res))
            dl = torch.rand((w.n_views, w.res, w.res), device="cuda") * 2 - 1
            g = P.CloudGrads(cloud.size())
            # capacity from one exact binning (sync-free steps, as bench.py), then the timed steps
            f = eng.render(cloud, sc, thetas)
            gpe, pairs = f.work()
            f.free()
            eng.set_capacity(int(pairs * 1.02) + 65536, 0)
            ev = []
            for k in range(a.steps + 1):
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                f = eng.render(cloud, sc, thetas)
                eng.render_backward(cloud, f, dl, g)
                e.record()
                f.free()
                ev.append((s, e))
            torch.cuda.synchronize()
            assert not eng.take_overflow()
            eng.set_capacity(0, 0)
            eng.set_timing(True)
            f = eng.render(cloud, sc, thetas)
            eng.render_backward(cloud, f, dl, g)
            f.free()
            kt = eng.timing_report()
            eng.set_timing(False)
            out["kernels_ms"] = {k: round(v[0], 3) for k, v in kt.items()}
            out["step_ms"] = [round(s.elapsed_time(e), 2) for s, e in ev]
            ms = float(np.median([s.elapsed_time(e) for s, e in ev[1:]]))
            out.update(views=w.n_views, res=w.res, ms_per_step=round(ms, 3), proj_per_s=round(w.n_views / ms * 1e3, 1),
                       pairs=pairs, gpe=gpe, grads_finite=bool(torch.isfinite(g.flat()).all().item()),
                       peak_mem_gb=round(torch.cuda.max_memory_allocated() / 1e9, 2))
        if a.voxel or not w.n_views:
            grid = P.grid_for_extent((-1, -1, -1), (1, 1, 1), (w.n_vox,) * 3)
            up = torch.rand(grid.shape_zyx, device="cuda") * 2 - 1
            g = P.CloudGrads(cloud.size())
            ev = []
            for k in range(a.steps + 1):
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                v = eng.voxelize(cloud, grid)
                eng.voxelize_backward(cloud, grid, up, g)
                e.record()
                ev.append((s, e))
            torch.cuda.synchronize()
            ms = float(np.median([s.elapsed_time(e) for s, e in ev[1:]]))
            out.update(voxel_ms=round(ms, 3), voxels_per_s=round(grid.voxel_count() / ms * 1e3),
                       vol_finite=bool(torch.isfinite(v).all().item()))
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
