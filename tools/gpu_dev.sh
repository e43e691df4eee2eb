#!/bin/bash
# development GPU pass: -m gpu suite, quick cfg3 bench, 8-rank shard probe, cfg2 train probe
cd ${GRAFT_REPO_ROOT:-.}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_dev.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest_dev.log
tail -3 gpurun_out/gputest_dev.log
STEPS=10 timeout 300 bash tools/quick_bench.sh
timeout 400 python tools/probe_shard.py 2>&1 | head -5
timeout 300 python tools/probe_train.py 2>&1 | tail -1
