cd $GRAFT_REPO_ROOT
for k in mma tc; do echo "== $k"; SCT_K4=$k STEPS=10 timeout 300 bash tools/quick_bench.sh; done > gpurun_out/k4cmp.log 2>&1
for i in 1 2 3 4 5; do SCT_K4=tc timeout 60 python -m pytest tests/test_gpu_parity.py -x -q -k "host_entry" 2>&1 | tail -2; echo rc=$?; done > gpurun_out/hu_loop.log 2>&1
for i in 1 2 3; do SCT_K4=mma timeout 60 python -m pytest tests/test_gpu_parity.py -x -q -k "host_entry" 2>&1 | tail -2; done >> gpurun_out/hu_loop.log 2>&1
