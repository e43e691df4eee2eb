"""Per-call wall time of the host-buffer entry points at cfg3 (diagnostic)."""
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_20693_b200 as P  # noqa: E402
from paper_2405_20693_b200 import _capi, scenes  # noqa: E402

ca = scenes.make_cloud(3)
eng = P.Engine(0)
L = _capi.load()
if os.environ.get("ATOMIC"):
    L.sct_ctx_set_deterministic(eng._h, 0)
thetas = [2 * np.pi * i / 75 for i in range(75)]
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
host = {k: pin(getattr(ca, k)) for k in ("rho_raw", "pos", "scale_raw", "rot")}
cl = _capi.sct_cloud()
cl.m, cl.s_min_mm = ca.m, ca.s_min
for k, t in host.items():
    setattr(cl, k, t.data_ptr())
imgs = torch.empty((75, 512, 512), dtype=torch.float32).pin_memory()
dL = torch.rand((75, 512, 512), dtype=torch.float32).pin_memory()
gbuf = torch.zeros(11 * ca.m, dtype=torch.float32).pin_memory()
parts = torch.split(gbuf, [ca.m, 3 * ca.m, 3 * ca.m, 4 * ca.m])
g = _capi.sct_grads()
for k, t in zip(("rho_raw", "pos", "scale_raw", "rot"), parts):
    setattr(g, k, t.data_ptr())
sc = P.ScannerConfig(detector_res_px=(512, 512))._c()
op = P.RasterOptions()._c()
th = (C.c_double * 75)(*thetas)
res = []
for it in range(15):
    st = C.c_void_p()
    t0 = time.perf_counter()
    assert L.sct_render_fwd_host(eng._h, C.byref(cl), C.byref(sc), th, 75, C.byref(op),
                                 C.c_void_p(imgs.data_ptr()), C.byref(st)) == 0
    t1 = time.perf_counter()
    assert L.sct_render_bwd_host(eng._h, st, C.byref(cl), C.c_void_p(dL.data_ptr()), C.byref(g), None) == 0
    t2 = time.perf_counter()
    L.sct_fwd_free(st)
    res.append((round(1e3 * (t1 - t0), 2), round(1e3 * (t2 - t1), 2)))
print(os.environ.get("SCT_HOST_UNITS", "1"), os.environ.get("SCT_HOST_CHUNKS", "auto"), res[3:])
