#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}
for p in 0 2 4 8 16; do echo -n "parts=$p "; SCT_K4_PARTS=$p timeout 300 python tools/probe_train.py 2>&1 | grep -E "K4_backward|wall without" | tr '\n' ' '; echo; done
