#!/bin/bash
# ncu evidence for profiles/ (round 2). Each capture runs only after the same
# command exited 0 without ncu. Reports are summarised on the box (they exceed
# what gpurun copies back); only the summaries and small reports return.
#   1. launch list of a short default bench run (per-launch durations)
#   2. hardware-unit metrics of one pass of every kernel family
#      (tools/profile_step.py: cfg3 raster fwd+bwd, cfg4 voxel fwd+bwd, cfg2
#      train iterations + adaptive control) -> tools/hw_units.py
#   3. the same for the FP32 SIMT arms of K4 / K8 (SCT_K4=simt SCT_K8=simt)
#   4. --set full of the two hottest raster kernels (K3, K4) -> ncu_summary
TAG=${1:-r02}
O=gpurun_out
B="python bench.py --no-cpu --no-e2e --no-simt-arm --steps 2 --warmup 3"
$B > $O/plain_$TAG.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$TAG.csv $B > $O/ncu_launch_$TAG.log 2>&1
python tools/launch_shares.py $O/launches_$TAG.csv > $O/launch_shares_$TAG.txt
M=sm__inst_issued.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed.sum.per_cycle_elapsed,sm__cycles_elapsed.avg.per_second,sm__warps_active.avg.pct_of_peak_sustained_active
P="python tools/profile_step.py"
$P > /dev/null 2>&1 || exit 1
ncu --metrics $M --clock-control none --profile-from-start off -o $O/units_$TAG -f $P > $O/ncu_units_$TAG.log 2>&1
python tools/hw_units.py $O/units_$TAG.ncu-rep > $O/hw_units_$TAG.json
SCT_K4=simt SCT_K8=simt $P --parts raster,voxel > /dev/null 2>&1 || exit 1
SCT_K4=simt SCT_K8=simt ncu --metrics $M --clock-control none --profile-from-start off -o $O/units_simt_$TAG -f $P --parts raster,voxel > $O/ncu_units_simt_$TAG.log 2>&1
python tools/hw_units.py $O/units_simt_$TAG.ncu-rep > $O/hw_units_simt_$TAG.json
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"composite_kernel|backward_stats_mma_kernel" -c 2 -o $O/full_$TAG -f $P --parts raster > $O/ncu_full_$TAG.log 2>&1
python tools/ncu_summary.py $O/full_$TAG.ncu-rep > $O/ncu_full_$TAG.txt
for f in $O/*.ncu-rep; do [ $(stat -c %s $f) -gt 30000000 ] && rm -f $f; done
ls -la $O
