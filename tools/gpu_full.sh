#!/bin/bash
# GPU round check: -m gpu suite, smoke, then the default bench (JSON line -> gpurun_out/bench_$TAG.json)
TAG=${1:-dev}
cd ${GRAFT_REPO_ROOT:-.}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest_$TAG.log
tail -3 gpurun_out/gputest_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; tail -1 gpurun_out/smoke_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
tail -c 600 gpurun_out/bench_$TAG.err
