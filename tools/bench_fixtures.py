"""Times device fixture generation at the cfg3 scale:
phantom 256^3, quadrature projections 75 x 512^2 (step = half a voxel),
host noise, FDK 256^3, init cloud 100k (NN distances + sampling)."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2405_20693_b200 as P
from paper_2405_20693_b200 import simulate as S


def timed(fn, reps=1):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        out = fn()
    torch.cuda.synchronize()
    return out, (time.perf_counter() - t0) / reps * 1e3


def main():
    eng = P.default_engine()
    n, res, views, m = 256, 512, 75, 100000
    th = P.full_circle_angles(views)
    cfg = P.ScannerConfig(detector_res_px=(res, res))
    S.phantom_shepp_logan_3d((32, 32, 32))  # warm-up
    (ph, grid), t_ph = timed(lambda: S.phantom_shepp_logan_3d((n, n, n)))
    step = 0.5 * grid.spacing_mm[0]
    clean, t_proj = timed(lambda: S.project_volume(ph, grid, cfg, th, step))
    noisy, t_noise = timed(lambda: S.add_noise(clean, S.NoiseParams(seed=7)))
    noisy = noisy.cuda()
    vol, t_fdk = timed(lambda: S.fdk_reconstruct(noisy, cfg, th, grid))
    cloud, t_init = timed(lambda: S.sample_init_cloud(ph, grid, m, seed=0))
    pts = cloud.pos.double().reshape(-1, 3)
    _, t_nn = timed(lambda: S.nearest_neighbor_distances(pts))
    samples = views * res * res * (2.0 * 1.5 / step)  # upper bound on trilinear samples
    print(json.dumps({
        "workload": f"{n}^3 phantom, {views} views at {res}^2, {m} kernels",
        "phantom_ms": t_ph, "project_volume_ms": t_proj, "noise_host_ms": t_noise, "fdk_ms": t_fdk,
        "sample_init_ms": t_init, "nn_distances_ms": t_nn,
        "fdk_psnr_vs_phantom_db": float(10 * torch.log10(1 / ((vol.clamp(0, 1) - ph) ** 2).mean())),
    }))


if __name__ == "__main__":
    main()
