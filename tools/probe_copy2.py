"""H2D / D2H bandwidth of pinned copies: one stream vs several concurrent streams."""
import time

import torch

n = 75 * 512 * 512
x = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty_like(x, device="cuda")
for ns in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    parts = [(i * n // ns, (i + 1) * n // ns) for i in range(ns)]
    for direction in ("H2D", "D2H"):
        for _ in range(3):
            for s, (a, b) in zip(streams, parts):
                with torch.cuda.stream(s):
                    (d[a:b].copy_(x[a:b], non_blocking=True) if direction == "H2D"
                     else x[a:b].copy_(d[a:b], non_blocking=True))
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(10):
            for s, (a, b) in zip(streams, parts):
                with torch.cuda.stream(s):
                    (d[a:b].copy_(x[a:b], non_blocking=True) if direction == "H2D"
                     else x[a:b].copy_(d[a:b], non_blocking=True))
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t) / 10
        print(f"{ns} stream(s) {direction} {n * 4 / dt / 1e9:.1f} GB/s")
