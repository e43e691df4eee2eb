"""Times the host-buffer C-ABI entry points piecewise at cfg3 (diagnostic)."""
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
eng = P.Engine(0, deterministic=os.environ.get("PROBE_DETERMINISTIC") == "1")  # bench.py: atomic
L = _capi.load()
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
for it in range(4):
    st = C.c_void_p()
    t0 = time.perf_counter()
    L.sct_render_fwd_host(eng._h, C.byref(cl), C.byref(sc), th, 75, C.byref(op), C.c_void_p(imgs.data_ptr()),
                          C.byref(st))
    t1 = time.perf_counter()
    L.sct_render_bwd_host(eng._h, st, C.byref(cl), C.c_void_p(dL.data_ptr()), C.byref(g), None)
    t2 = time.perf_counter()
    L.sct_fwd_free(st)
    print(f"fwd_host {1e3*(t1-t0):.2f} ms  bwd_host {1e3*(t2-t1):.2f} ms")
# device path for comparison
cloud = P.GaussianCloud(ca.s_min, ca.rho_raw, ca.pos, ca.scale_raw, ca.rot)
dd = dL.cuda()
gr = P.CloudGrads(ca.m)
scn = P.ScannerConfig(detector_res_px=(512, 512))
for it in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    f = eng.render(cloud, scn, thetas)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    eng.render_backward(cloud, f, dd, gr)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    f.free()
    print(f"device fwd {1e3*(t1-t0):.2f} ms  bwd {1e3*(t2-t1):.2f} ms")
x = torch.empty(75 * 512 * 512, device="cuda")
torch.cuda.synchronize()
t0 = time.perf_counter()
x.copy_(dL.view(-1), non_blocking=True)
torch.cuda.synchronize()
print(f"torch H2D 78.6MB {1e3*(time.perf_counter()-t0):.2f} ms")
for _ in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    imgs.view(-1).copy_(x, non_blocking=True)
    torch.cuda.synchronize()
    print(f"torch D2H 78.6MB {1e3*(time.perf_counter()-t0):.2f} ms")

# long loops: per-step wall times of the host path and the device path
import subprocess
smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active",
                        "--format=csv,noheader", "-lms", "100"], stdout=subprocess.PIPE, text=True)
hw = []
for it in range(30):
    st = C.c_void_p()
    t0 = time.perf_counter()
    L.sct_render_fwd_host(eng._h, C.byref(cl), C.byref(sc), th, 75, C.byref(op), C.c_void_p(imgs.data_ptr()),
                          C.byref(st))
    L.sct_render_bwd_host(eng._h, st, C.byref(cl), C.c_void_p(dL.data_ptr()), C.byref(g), None)
    L.sct_fwd_free(st)
    hw.append(round(1e3 * (time.perf_counter() - t0), 1))
print("host path per step ms:", hw)
dw = []
for it in range(30):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    f = eng.render(cloud, scn, thetas)
    eng.render_backward(cloud, f, dd, gr)
    f.free()
    torch.cuda.synchronize()
    dw.append(round(1e3 * (time.perf_counter() - t0), 1))
print("device path per step ms:", dw)
smi.terminate()
out = smi.communicate()[0].strip().splitlines()
print("smi samples:", len(out), out[:3], out[-3:])
