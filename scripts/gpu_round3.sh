#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -15
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_serial -s 0 -c 1 -o gpurun_out/serial_r3 python scripts/gpu_diff.py c2 20000 > gpurun_out/ncu_serial3.log 2>&1; tail -1 gpurun_out/ncu_serial3.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_match -s 1 -c 1 -o gpurun_out/match_r3 python scripts/gpu_diff.py c2 40000 > gpurun_out/ncu_match3.log 2>&1; tail -1 gpurun_out/ncu_match3.log
