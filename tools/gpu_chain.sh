#!/bin/bash
# K5 chain layout sweep (SCT_CHAIN_LANES) on the quick cfg3 bench
cd ${GRAFT_REPO_ROOT:-.}
for l in 1 2 4 16; do echo -n "lanes=$l "; SCT_CHAIN_LANES=$l STEPS=10 bash tools/quick_bench.sh; done
timeout 300 python tools/probe_train.py
