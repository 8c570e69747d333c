#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -5
timeout 600 python bench.py --steps 3 --warmup 1 > gpurun_out/bench5.json 2>gpurun_out/bench5.err; tail -c 1500 gpurun_out/bench5.json; tail -3 gpurun_out/bench5.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_serial -s 0 -c 1 -o gpurun_out/serial_r5 python scripts/gpu_diff.py c2 20000 > gpurun_out/ncu_serial5.log 2>&1; tail -1 gpurun_out/ncu_serial5.log
