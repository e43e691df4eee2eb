"""List-length distribution of the cfg3 forward (diagnostic for K3/K4 tails)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2405_20693_b200 as P  # noqa: E402

w, ca, thetas, vol = bench.make_workload()
eng = P.Engine(0)
cloud = P.GaussianCloud(ca.s_min, ca.rho_raw, ca.pos, ca.scale_raw, ca.rot, device="cuda")
scanner = P.ScannerConfig(detector_res_px=(w.res, w.res))
f = eng.render(cloud, scanner, thetas)
lens = []
for v in (0, 18, 37):
    off, _ = f.tile_lists(v)
    lens.append(np.diff(off))
L = np.concatenate(lens)
tot = L.sum()
print("tiles", L.size, "pairs", tot, "mean", L.mean(), "max", L.max(), "p99", np.percentile(L, 99), "p90", np.percentile(L, 90))
s = np.sort(L)[::-1]
print("top10", s[:10].tolist())
print("work share of lists > 4x mean", s[s > 4 * L.mean()].sum() / tot, "count", (s > 4 * L.mean()).sum())
