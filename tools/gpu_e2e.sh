#!/bin/bash
# host-path checks: the host-entry GPU tests, then cfg3 device / e2e rates with and without the split forward
cd ${GRAFT_REPO_ROOT:-.}
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_host_fallback.py tests/test_gpu_io.py -x -q -k "host" 2>&1 | tail -3
for sp in 1 0; do echo -n "split=$sp "; SCT_HOST_SPLIT=$sp timeout 300 python bench.py --no-cpu --no-voxel --no-train --no-simt-arm --steps 10 2>/tmp/e2e_err.log | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']), round(d['e2e']['value']), round(d['e2e']['ms_per_step'],3), round(d['e2e']['per_view_calls']['value']))"; grep "fwd_host" /tmp/e2e_err.log | cut -c1-200; done
