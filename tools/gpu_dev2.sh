#!/bin/bash
# development GPU pass: -m gpu suite, quick cfg3 bench, voxel K7/K8 times, cfg2 train probe
cd ${GRAFT_REPO_ROOT:-.}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_dev.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest_dev.log
tail -3 gpurun_out/gputest_dev.log
STEPS=10 timeout 300 bash tools/quick_bench.sh
timeout 300 python bench.py --no-cpu --no-e2e --no-train --no-simt-arm --steps 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); v=d['voxelizer']; print('voxel', round(v['value']/1e9,2), {k: round(x['ms_per_step'],3) for k,x in v['kernels'].items()})"
timeout 300 python tools/probe_train.py 2>&1 | tail -1
