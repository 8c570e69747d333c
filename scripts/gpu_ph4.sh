#!/bin/bash
# dev: per-phase cycles on C4 / C2 / C1 (E2_PHASES build in build/)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in ${PH_CONFIGS:-c4:100000 c2:30000 c1:1000}; do timeout 600 python scripts/phases.py build/libe2phases.so ${c%%:*} ${c##*:} 2>&1 | tail -1; done
