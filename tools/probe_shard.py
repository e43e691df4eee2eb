"""Per-rank step time of the cfg3 workload when the 75 views are sharded over
N ranks (strong scaling), measured on one GPU by running rank 0's shard: the
compute side of the N-GPU step (the NCCL all-reduce of 11*M floats is extra)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2405_20693_b200 as P  # noqa: E402
from paper_2405_20693_b200 import dist as pdist  # noqa: E402

w, ca, thetas, vol = bench.make_workload()
eng = P.Engine(0, deterministic=False)
cloud = P.GaussianCloud(ca.s_min, ca.rho_raw, ca.pos, ca.scale_raw, ca.rot, device="cuda")
scanner = P.ScannerConfig(detector_res_px=(w.res, w.res))
grads = P.CloudGrads(cloud.size())
t1 = None
for world in (1, 2, 4, 8):
    views = pdist.shard_views(len(thetas), 0, world)
    th = [thetas[v] for v in views]
    dL = torch.from_numpy(bench.upstream(len(thetas), w.res, views)).cuda()
    imgs = torch.empty((len(th), w.res, w.res), device="cuda")

    def step():
        grads.zero_()
        f = eng.render(cloud, scanner, th, out=imgs)
        eng.render_backward(cloud, f, dL, grads)
        f.free()

    eng.set_capacity(0, 0)
    step()
    f = eng.render(cloud, scanner, th, out=imgs)
    n_pairs = f.work()[1]
    f.free()
    eng.set_capacity(int(n_pairs * 1.02) + 65536, 0)  # sync-free binning, as bench.py
    for _ in range(8):
        step()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(20):
        step()
    ev[1].record()
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1]) / 20
    t1 = t1 or ms
    print(f"N={world}: rank-0 shard {len(th)} views, {ms:.3f} ms/step, ideal {t1 / world:.3f}, "
          f"compute-side efficiency {t1 / world / ms:.2f}")

# kernel breakdown of the N=8 shard (engine timing events; adds per-launch overhead)
views = pdist.shard_views(len(thetas), 0, 8)
th = [thetas[v] for v in views]
dL = torch.from_numpy(bench.upstream(len(thetas), w.res, views)).cuda()
imgs = torch.empty((len(th), w.res, w.res), device="cuda")
eng.set_timing(True)
for _ in range(10):
    grads.zero_()
    f = eng.render(cloud, scanner, th, out=imgs)
    eng.render_backward(cloud, f, dL, grads)
    f.free()
torch.cuda.synchronize()
rep = eng.timing_report()
eng.set_timing(False)
for k, v in sorted(rep.items(), key=lambda kv: -kv[1][0]):
    print(f"  {k:28s} {v[0] / 10 * 1e3:8.1f} us  x{v[1] / 10:.1f}")
