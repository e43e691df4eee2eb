#!/bin/bash
# Round-2 evidence pass: full default bench, profile_round2.sh (launch list,
# hardware units, SIMT arm units, K3/K4 --set full), bench_configs cfg1/cfg5
TAG=${1:-r02d}
cd ${GRAFT_REPO_ROOT:-.}
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_$TAG.json 2>/dev/null; echo "ref rc=$?"
timeout 1500 bash tools/profile_round2.sh $TAG > gpurun_out/prof_$TAG.log 2>&1; echo "prof rc=$?"
timeout 900 python tools/bench_configs.py --config 1 5 --voxel --steps 6 > gpurun_out/configs_$TAG.jsonl 2> gpurun_out/configs_$TAG.err; echo "configs rc=$?"
ls gpurun_out
