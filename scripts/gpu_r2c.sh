#!/bin/bash
# round 2 first look: GPU tests, all configs (C4 shape), bench line on C4 + reference arm
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
nproc
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_r2c.log 2>&1; tail -3 gpurun_out/pytest_r2c.log
timeout 1500 python scripts/configs_report.py c4 c1 c2 c3 > gpurun_out/configs_r2c.jsonl 2>&1; cut -c1-700 gpurun_out/configs_r2c.jsonl
timeout 1500 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_r2c.json 2>gpurun_out/bench_r2c.err; tail -c 3000 gpurun_out/bench_r2c.json; tail -3 gpurun_out/bench_r2c.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_r2c.json 2>&1; tail -c 800 gpurun_out/bench_ref_r2c.json
