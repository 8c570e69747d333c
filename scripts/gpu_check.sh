#!/bin/bash
# dev: full GPU check — tests, bench line, all-config report, launch list
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
tag=${1:-x}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_$tag.log 2>&1; tail -5 gpurun_out/pytest_$tag.log
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_$tag.json 2>gpurun_out/bench_$tag.err; tail -c 2500 gpurun_out/bench_$tag.json; tail -3 gpurun_out/bench_$tag.err
timeout 900 python scripts/configs_report.py > gpurun_out/configs_$tag.jsonl 2>&1; cat gpurun_out/configs_$tag.jsonl | cut -c1-600
