#!/usr/bin/env python
"""Per-kernel share of device time from an ncu `--metrics gpu__time_duration.sum --csv` launch list.
ncu's per-launch times are cold-cache and serialised: compare SHARES, not absolute times."""
import csv
import sys
from collections import defaultdict


def main(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[hdr + 1:]:
        name = r[ki].split("(")[0].replace("sct::<unnamed>::", "").replace("void ", "")[:70]
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}.get(r[ui], 1e-6)
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", "")) * scale
    tot = sum(v[1] for v in agg.values())
    print(f"{'total ms':>10s} {'share':>6s} {'launches':>8s}  kernel   (source: {path})")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{v[1]:10.3f} {100 * v[1] / tot:5.1f}% {v[0]:8d}  {k}")


if __name__ == "__main__":
    main(sys.argv[1])
