"""Relative L2 error of the render_backward gradients against the FP64 oracle
on the golden fixtures, for the K4 variant selected by SCT_K4."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_20693_b200 as P  # noqa: E402
from tests import _golden as G  # noqa: E402
from tests._helpers import rel_l2  # noqa: E402

out = {}
for det in (True, False):
    for name in ("rectified", "biased_frozen_nolp"):
        s_min, *arrs = G.cloud_arrays()
        c = P.GaussianCloud(s_min, *arrs)
        eng = P.Engine(0, deterministic=det)
        man, imgs, dL, z = G.raster(name)
        w, h = man["raster"]["res"]
        fwd = eng.render(c, P.ScannerConfig(detector_res_px=(w, h)), man["raster"]["thetas"],
                         P.RasterOptions(**man["option_sets"][name]))
        g = P.CloudGrads(c.size())
        eng.render_backward(c, fwd, torch.from_numpy(dL).cuda(), g, accumulate_stats=True)
        torch.cuda.synchronize()
        errs = {k: rel_l2(getattr(g, k).cpu().numpy(), z["g_" + k]) for k in ("rho_raw", "pos", "scale_raw", "rot")}
        errs["norm"] = rel_l2(c.grad2d_norm_accum.cpu().numpy(), z["grad2d_norm_accum"])
        out[f"{name}/{'det' if det else 'atomic'}"] = {k: float(f"{v:.2e}") for k, v in errs.items()}
print(os.environ.get("SCT_K4", "default"), out)
