#!/bin/bash
# round-2 first look: GPU tests + all configs (new C4 shape) on the B200
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
nproc
timeout 1500 python scripts/configs_report.py c4 c1 c2 c3 > gpurun_out/configs_r2a.jsonl 2>&1; cut -c1-900 gpurun_out/configs_r2a.jsonl
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_r2a.log 2>&1; tail -3 gpurun_out/pytest_r2a.log
