#!/bin/bash
# short cfg3 bench: headline value + per-kernel ms (no CPU / e2e / voxel / train legs)
python bench.py --no-cpu --no-e2e --no-voxel --no-train --steps ${STEPS:-8} --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']), {k: round(v['ms_per_step'],3) for k,v in d['kernels'].items()})"
