"""Where a cfg2 train iteration spends its time: device kernel sum vs wall."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_20693_b200 as P  # noqa: E402
from paper_2405_20693_b200 import scenes  # noqa: E402
from paper_2405_20693_b200.train import TrainConfig, Trainer  # noqa: E402

eng = P.Engine(0)
w = scenes.CONFIGS[2]
ca = scenes.make_cloud(2)
angles = P.full_circle_angles(w.n_views)
sc = P.ScannerConfig(detector_res_px=(w.res, w.res))
f = eng.render(P.GaussianCloud(ca.s_min, ca.rho_raw, ca.pos, ca.scale_raw, ca.rot), sc, angles)
meas = f.images.clone()
f.free()
cloud = P.GaussianCloud(ca.s_min, ca.rho_raw, ca.pos, ca.scale_raw, ca.rot)
tr = Trainer(eng, cloud, sc, angles, meas, TrainConfig(iters=1000, output_dims=(w.n_vox,) * 3, check_every=0))
for _ in range(20):
    tr.step()
torch.cuda.synchronize()
eng.set_timing(True)
n = 50
t0 = time.perf_counter()
for _ in range(n):
    tr.step()
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / n * 1e3
rep = eng.timing_report()
eng.set_timing(False)
tot = sum(v[0] for v in rep.values()) / n
print(f"wall {wall:.3f} ms/iter, engine kernels {tot:.3f} ms/iter, launches {sum(v[1] for v in rep.values()) / n:.0f}")
for k, v in sorted(rep.items(), key=lambda kv: -kv[1][0]):
    print(f"  {k:28s} {v[0] / n * 1e3:8.1f} us  x{v[1] / n:.1f}")
t0 = time.perf_counter()
for _ in range(n):
    tr.step()
torch.cuda.synchronize()
print(f"wall without timing {(time.perf_counter() - t0) / n * 1e3:.3f} ms/iter")
