#!/bin/bash
# round 2: GPU tests after the replay refactor + per-phase cycles on C4/C2/C1
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_r2d.log 2>&1; tail -3 gpurun_out/pytest_r2d.log
for c in c4:100000 c2:30000 c1:1000; do timeout 600 python scripts/phases.py build/libe2phases.so ${c%%:*} ${c##*:} 2>&1 | tail -1; done > gpurun_out/phases_r2d.txt; cat gpurun_out/phases_r2d.txt
