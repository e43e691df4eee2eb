#!/usr/bin/env python
"""Per-kernel hardware-unit utilisation from an `ncu --set full` report: the
binding unit (the busiest of issue slots, FP32 FMA pipe, FP64 pipe, XU/MUFU,
tensor pipe, L1/shared LSU wavefronts, L2, DRAM) and its fraction, DRAM bytes
and executed thread-instructions. Launches of the same kernel are summed /
duration-weighted.  Usage: python tools/hw_units.py report.ncu-rep > out.json"""
import csv
import io
import json
import subprocess
import sys
from collections import OrderedDict

UNITS = OrderedDict([
    ("issue_slots", "sm__inst_issued.avg.pct_of_peak_sustained_active"),
    ("fp32_fma_pipe", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
    ("fp64_pipe", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
    ("xu_mufu", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
    ("alu", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
    ("tensor_pipe", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
    ("l1_lsu_wavefronts", "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"),
    ("l2", "lts__throughput.avg.pct_of_peak_sustained_elapsed"),
])
HBM_PEAK_GBS = 6546.2  # MEASURED_PEAKS.json hbm_gbs (copy bandwidth)
EXTRA = {"duration_ns": "gpu__time_duration.sum", "dram_read": "dram__bytes_read.sum",
         "dram_write": "dram__bytes_write.sum", "ipc_elapsed": "sm__inst_executed.sum.per_cycle_elapsed",
         "sm_mhz": "sm__cycles_elapsed.avg.per_second",
         "occupancy_pct": "sm__warps_active.avg.pct_of_peak_sustained_active"}


def to_float(v):
    try:
        return float(v.replace(",", ""))
    except Exception:
        return None


def scale(unit):
    return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3, "msecond": 1e6,
            "ns": 1, "us": 1e3, "ms": 1e6, "s": 1e9, "hz": 1e-6, "Khz": 1e-3, "Mhz": 1, "Ghz": 1e3}.get(unit, 1)


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    col = {name: j for j, name in enumerate(h)}
    agg = OrderedDict()
    for r in rows[2:]:
        name = r[col["Kernel Name"]].replace("<unnamed>::", "").replace("(anonymous namespace)::", "")
        name = name.split("(")[0].replace("void ", "").strip()
        if "<" in name:  # template arguments: keep the first one (e.g. raster_chain_kernel<0>)
            name = name.split("<")[0] + "<" + name.split("<")[1].split(",")[0].split(">")[0] + ">"
        name = name.split("::")[-1] if "::" in name.split("<")[0] else name
        d = agg.setdefault(name, {"launches": 0, "w": 0.0, "units": {k: 0.0 for k in UNITS},
                                  **{k: 0.0 for k in EXTRA}, "warp_inst": 0.0})
        vals = {}
        for k, m in EXTRA.items():
            if m in col:
                x = to_float(r[col[m]])
                vals[k] = None if x is None else x * scale(u[col[m]])
        dur = vals.get("duration_ns") or 0.0
        d["launches"] += 1
        d["w"] += dur
        for k in ("duration_ns", "dram_read", "dram_write"):
            d[k] += vals.get(k) or 0.0
        # warp instructions = SM-summed IPC x elapsed cycles
        d["warp_inst"] = d.get("warp_inst", 0.0) + (vals.get("ipc_elapsed") or 0.0) * dur * (vals.get("sm_mhz") or 0.0) * 1e-3
        d["sm_mhz"] += (vals.get("sm_mhz") or 0.0) * dur
        d["occupancy_pct"] += (vals.get("occupancy_pct") or 0.0) * dur
        for k, m in UNITS.items():
            x = to_float(r[col[m]]) if m in col else None
            d["units"][k] += (x or 0.0) * dur
    res = OrderedDict()
    for name, d in agg.items():
        w = d["w"] or 1.0
        units = {k: round(v / w / 100.0, 4) for k, v in d["units"].items()}
        units["dram"] = round((d["dram_read"] + d["dram_write"]) / (d["duration_ns"] or 1.0) / HBM_PEAK_GBS, 4)
        bound = max(units, key=units.get)
        n = d["launches"]
        res[name] = {"launches": n, "ncu_us_per_launch": round(d["duration_ns"] / n / 1e3, 2),
                     "sm_mhz": round(d["sm_mhz"] / w, 0), "occupancy": round(d["occupancy_pct"] / w / 100.0, 3),
                     "bound_unit": bound, "bound_frac": units[bound], "units": units,
                     "dram_bytes_per_launch": int((d["dram_read"] + d["dram_write"]) / n),
                     "dram_gbs_under_ncu": round((d["dram_read"] + d["dram_write"]) / (d["duration_ns"] or 1), 1),
                     "warp_inst_per_launch": int(d["warp_inst"] / n)}
    json.dump(res, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main(sys.argv[1])
