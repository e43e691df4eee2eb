#!/bin/bash
# development GPU pass: -m gpu suite, quick cfg3 bench, 8-rank shard probe, cfg2 train
cd ${GRAFT_REPO_ROOT:-.}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_dev.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest_dev.log
tail -3 gpurun_out/gputest_dev.log
STEPS=10 timeout 300 bash tools/quick_bench.sh
timeout 500 python tools/probe_shard.py 2>&1 | tail -17
timeout 300 python bench.py --no-cpu --no-e2e --no-voxel --no-simt-arm --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg3', round(d['value']), 'train', round(d['train_step']['value']))"
