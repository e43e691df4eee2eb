#!/bin/bash
# K4 variant comparison (SCT_K4=mma|tc|simt; round 1 also had tf32 forms, since removed):
# parity error on the golden fixtures + cfg3 K4 time.
for v in ${VARIANTS:-mma tc simt}; do
  SCT_K4=$v python tools/probe_k4_precision.py
  SCT_K4=$v python bench.py --no-cpu --no-e2e --no-voxel --no-train --steps 5 --warmup 3 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['value']), {k: round(v['ms_per_step'],3) for k,v in d['kernels'].items() if k.startswith('K4') or k.startswith('K5_raster_chain')})"
done
