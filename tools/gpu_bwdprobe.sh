#!/bin/bash
# host-path backward timeline variants (SCT_UNIT_DEBUG marks)
cd ${GRAFT_REPO_ROOT:-.}
for g in 1 2; do echo "== chain groups $g"; SCT_CHAIN_GROUPS=$g SCT_UNIT_DEBUG=1 timeout 300 python tools/probe_e2e.py 2>&1 | grep "bwd_host\]" | tail -2; done
echo "== no host units (chunked)"; SCT_HOST_UNITS=0 timeout 300 python tools/probe_e2e.py 2>&1 | grep "^fwd_host" | tail -2
