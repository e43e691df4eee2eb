#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}
for w in 2 4; do echo "== SCT_K4_W=$w"; SCT_K4_W=$w timeout 400 python tools/probe_shard.py 2>&1 | head -4; done
echo "== default"; timeout 400 python tools/probe_shard.py 2>&1 | head -4
