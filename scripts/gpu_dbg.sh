#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/dbg_deep.py 2>&1 | tail -3
timeout 600 compute-sanitizer --tool memcheck --print-limit 10 python scripts/dbg_deep.py > gpurun_out/dbg_memcheck.log 2>&1; grep -v "^=========     " gpurun_out/dbg_memcheck.log | tail -4
timeout 1800 python -m pytest tests -x -q -m gpu --durations=15 > gpurun_out/pytest_r2h.log 2>&1; tail -22 gpurun_out/pytest_r2h.log
