import sys, numpy as np, torch
sys.path.insert(0, '.')
from oracle import oracle as O
import paper_2405_20693_b200 as P
from paper_2405_20693_b200.train import NativeTrainer, TrainConfig, Trainer
res, n_views = 64, 6
scanner_o = O.test_scanner(res)
angles = O.full_circle_angles(n_views)
target = O.random_cloud(O.Rng(5), 80, 0.6, 0.05, 0.15)
meas = torch.from_numpy(np.stack([O.render(target, scanner_o, th).image for th in angles]).astype(np.float32))
oc = O.random_cloud(O.Rng(7), 300, 0.6, 0.01, 0.12)
f32 = [np.asarray(a, dtype=np.float32) for a in (oc.rho_raw, oc.pos, oc.scale_raw, oc.rot)]
cfg = TrainConfig(iters=40, output_dims=(32, 32, 32), tv_grid_dim=8, adaptive_start=3, densify_interval=4,
                  densify_grad_threshold=1e-6, prune_density_threshold=0.05, seed=13, sync_free=True, check_every=1)
sc = P.ScannerConfig(detector_res_px=(res, res))
tr = Trainer(P.Engine(0), P.GaussianCloud(oc.s_min, *f32), sc, angles, meas, cfg)
nt = NativeTrainer(P.Engine(0), P.GaussianCloud(oc.s_min, *f32), sc, angles, meas, cfg)
for i in range(4):
    out = tr.step(); nt.step(); r = nt.record(); st = nt.state(); c = tr.cloud
    d = {k: float(np.abs(st[k].astype(np.float64) - getattr(c, k).cpu().numpy()).max()) for k in ("rho_raw","pos","scale_raw","rot","grad2d_norm_accum","grad3d_accum")}
    d["grad_count"] = int((st["grad_count"] != c.grad_count.cpu().numpy()).sum())
    print(i, out["view"], r["view"], float(out["l1"]) - r["l1"], float(out["tv"]) - r["tv"], d)
