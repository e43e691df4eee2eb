#!/bin/bash
# ncu --set full (+ source) of one launch of the kernels matching REGEX in one
# profiled cfg3 raster pass (tools/profile_step.py), after the same command ran
# clean without ncu; summary -> gpurun_out/ncu_$TAG.txt
REGEX=$1; TAG=$2; PARTS=${3:-raster}
cd ${GRAFT_REPO_ROOT:-.}
P="python tools/profile_step.py --parts $PARTS"
$P > /dev/null 2>&1 || { echo "plain run failed"; exit 1; }
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"$REGEX" -c ${COUNT:-1} \
    -o gpurun_out/$TAG -f $P > gpurun_out/ncu_$TAG.log 2>&1
python tools/ncu_summary.py gpurun_out/$TAG.ncu-rep > gpurun_out/ncu_$TAG.txt
tail -3 gpurun_out/ncu_$TAG.log
