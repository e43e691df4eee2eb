"""Host-side timing of the cfg3 step (diagnoses GPU bubbles caused by the host)."""
import os
import sys
import time

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
for _ in range(3):
    f = eng.render(cloud, scanner, thetas, out=images)
    eng.render_backward(cloud, f, dL, grads)
    f.free()
torch.cuda.synchronize()
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
host = []
for k in range(20):
    t0 = time.perf_counter()
    ev[k][0].record()
    grads.zero_()
    t1 = time.perf_counter()
    f = eng.render(cloud, scanner, thetas, out=images)
    t2 = time.perf_counter()
    eng.render_backward(cloud, f, dL, grads)
    t3 = time.perf_counter()
    ev[k][1].record()
    f.free()
    t4 = time.perf_counter()
    host.append((round((t1 - t0) * 1e3, 2), round((t2 - t1) * 1e3, 2), round((t3 - t2) * 1e3, 2), round((t4 - t3) * 1e3, 2)))
torch.cuda.synchronize()
for k in range(20):
    print(round(ev[k][0].elapsed_time(ev[k][1]), 3), host[k])
print("cpus", os.cpu_count(), "load", os.getloadavg())
