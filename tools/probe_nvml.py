"""Does in-process NVML sampling stall the device-resident step loop?"""
import os
import sys
import threading
import time

import pynvml
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2405_20693_b200 as P  # noqa: E402

w, ca, thetas, vol = bench.make_workload()
eng = P.Engine(0)
cloud = P.GaussianCloud(ca.s_min, ca.rho_raw, ca.pos, ca.scale_raw, ca.rot, device="cuda")
scanner = P.ScannerConfig(detector_res_px=(w.res, w.res))
dL = torch.from_numpy(bench.upstream(len(thetas), w.res, list(range(len(thetas))))).cuda()
grads = P.CloudGrads(cloud.size())
images = torch.empty((len(thetas), w.res, w.res), device="cuda")


def step():
    grads.zero_()
    f = eng.render(cloud, scanner, thetas, out=images)
    eng.render_backward(cloud, f, dL, grads)
    f.free()


for _ in range(15):
    step()
torch.cuda.synchronize()
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
for name, fns in [("none", []), ("clock", [lambda: pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)]),
                  ("reasons", [lambda: pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)]), ("none2", [])]:
    lat = []
    stop = [False]

    def loop():
        while not stop[0]:
            for f in fns:
                t = time.perf_counter()
                f()
                lat.append(time.perf_counter() - t)
            time.sleep(0.05)

    th = threading.Thread(target=loop, daemon=True)
    if fns:
        th.start()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
    for k in range(20):
        ev[k][0].record()
        step()
        ev[k][1].record()
    torch.cuda.synchronize()
    stop[0] = True
    if fns:
        th.join()
    st = [round(a.elapsed_time(b), 2) for a, b in ev]
    print(name, "steps", st, "nvml ms", [round(1e3 * x, 2) for x in lat][:10])
