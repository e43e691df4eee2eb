#!/bin/bash
# e2e (host-buffer path) vs the number of FP64 chain groups in the backward
cd ${GRAFT_REPO_ROOT:-.}
for g in 1 2 4; do echo -n "groups=$g "; SCT_CHAIN_GROUPS=$g timeout 300 python bench.py --no-cpu --no-voxel --no-train --no-simt-arm --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']), round(d['e2e']['value']), round(d['e2e']['ms_per_step'],3))"; done
