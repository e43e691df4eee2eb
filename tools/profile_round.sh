#!/bin/bash
# ncu evidence for profiles/: launch list of a short bench run (per-launch
# durations, clocks uncontrolled) and --set full captures of the hot raster and
# voxel kernels (all only after the same command exited 0 without ncu).
TAG=${1:-r01_v9}
CMD="python bench.py --no-cpu --no-e2e --no-train --steps 2 --warmup 3"
$CMD > gpurun_out/plain_$TAG.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"composite_kernel|backward_stats_mma_kernel|raster_chain_kernel|raster_preprocess_kernel" -s 12 -c 4 -o gpurun_out/prof_$TAG -f $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"voxel_eval_kernel|voxel_backward_mma_kernel|voxel_pair_sum_kernel|voxel_chain_kernel" -s 4 -c 4 -o gpurun_out/prof_vox_$TAG -f $CMD > gpurun_out/ncu_vox_$TAG.log 2>&1
