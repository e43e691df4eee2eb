#!/bin/bash
# one K4 launch of the selected variant at cfg3 under ncu --set full
export SCT_K4=${1:-tf32x2}
CMD="python bench.py --no-cpu --no-e2e --no-voxel --no-train --steps 1 --warmup 3"
$CMD > /dev/null 2>&1 && ncu --set full --import-source on -k regex:backward_stats -s 2 -c 1 -o gpurun_out/k4_$SCT_K4 -f $CMD > gpurun_out/k4_ncu_$SCT_K4.log 2>&1
