#!/bin/bash
# GPU check used during development: full -m gpu suite, then quick cfg3 benches of
# the product library and the named variants (tools/variants.sh).
cd ${GRAFT_REPO_ROOT:-.}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest.log
tail -3 gpurun_out/gputest.log
timeout 900 bash tools/variants.sh run base "$@" > gpurun_out/variants.log 2>&1
cat gpurun_out/variants.log
