#!/bin/bash
set -x
cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --steps 3 --warmup 1 2>&1 | tail -3
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/launches_r2.csv python bench.py --steps 1 --warmup 0 > gpurun_out/ncu_list.log 2>&1; tail -2 gpurun_out/ncu_list.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_serial -s 2 -c 1 -o gpurun_out/serial_r2 python scripts/gpu_diff.py c2 30000 > gpurun_out/ncu_serial.log 2>&1; tail -2 gpurun_out/ncu_serial.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_match -s 2 -c 1 -o gpurun_out/match_r2 python scripts/gpu_diff.py c2 30000 > gpurun_out/ncu_match.log 2>&1; tail -2 gpurun_out/ncu_match.log
