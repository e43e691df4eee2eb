#!/usr/bin/env python
"""Summarise an ncu report (details + raw pages) per kernel: duration, SOL
throughputs, occupancy, issue activity, pipe utilisation, DRAM bytes, stall
reasons. Usage: python tools/ncu_summary.py report.ncu-rep [> profiles/x.txt]"""
import csv
import io
import subprocess
import sys
from collections import OrderedDict

DETAILS = ["Duration", "SM Frequency", "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput",
           "Registers Per Thread", "Theoretical Occupancy", "Achieved Occupancy", "Executed Ipc Active",
           "Issue Slots Busy", "Eligible Warps Per Scheduler", "No Eligible", "Warp Cycles Per Issued Instruction",
           "L1/TEX Hit Rate", "L2 Hit Rate", "Block Limit Registers", "Block Limit Shared Mem", "Waves Per SM"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
       "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
       "sm__sass_thread_inst_executed_op_ffma_pred_on.sum", "sm__sass_thread_inst_executed_op_fadd_pred_on.sum",
       "sm__sass_thread_inst_executed_op_fmul_pred_on.sum"]
STALLS = "smsp__average_warp_latency_issue_stalled_"


def run(rep, page):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main(rep):
    rows = run(rep, "details")
    h = rows[0]
    ki, mi, vi, ui, idi = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    per = OrderedDict()
    for r in rows[1:]:
        key = (r[idi], r[ki].split("(")[0].replace("sct::<unnamed>::", "").replace("unnamed>::", ""))
        d = per.setdefault(key, {})
        if r[mi] in DETAILS and r[mi] not in d:
            d[r[mi]] = f"{r[vi]} {r[ui]}"
    raw = run(rep, "raw")
    rh, ru = raw[0], raw[1]
    rawper = {}
    for r in raw[2:]:
        rid = r[rh.index("ID")]
        d = {}
        for j, name in enumerate(rh):
            if name in RAW or name.startswith(STALLS):
                d[name] = f"{r[j]} {ru[j]}".strip()
        rawper[rid] = d
    for (rid, name), d in per.items():
        print(f"=== [{rid}] {name}")
        for k in DETAILS:
            if k in d:
                print(f"  {k:40s} {d[k]}")
        rd = rawper.get(rid, {})
        for k in RAW:
            if k in rd:
                print(f"  {k:70s} {rd[k]}")
        st = sorted(((float(v.split()[0].replace(',', '') or 0), k) for k, v in rd.items()
                     if k.startswith(STALLS) and v.split() and v.split()[0] not in ("", "n/a")), reverse=True)[:6]
        if st:
            print("  top stall reasons (avg warp latency, cycles):")
            for v, k in st:
                print(f"    {k[len(STALLS):]:50s} {v:.2f}")


if __name__ == "__main__":
    main(sys.argv[1])
