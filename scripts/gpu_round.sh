#!/bin/bash
# Round evidence: GPU tests, bench line, all-config report, ncu launch list of
# the bench command, one --set full capture each of k_serial and k_match.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
tag=${1:-r}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_$tag.log 2>&1; tail -3 gpurun_out/pytest_$tag.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_$tag.json 2>gpurun_out/bench_$tag.err; tail -c 3000 gpurun_out/bench_$tag.json; tail -2 gpurun_out/bench_$tag.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$tag.json 2>gpurun_out/bench_ref_$tag.err; tail -c 1500 gpurun_out/bench_ref_$tag.json
timeout 1500 python scripts/configs_report.py > gpurun_out/configs_$tag.jsonl 2>&1; cut -c1-700 gpurun_out/configs_$tag.jsonl
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv python bench.py --steps 1 --warmup 3 > gpurun_out/bench_ncu_$tag.log 2>&1; wc -l gpurun_out/launches_$tag.csv
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_serial -s 4 -c 1 -o gpurun_out/serial_$tag python scripts/gpu_diff.py c2 60000 > gpurun_out/ncu_serial_$tag.log 2>&1; tail -1 gpurun_out/ncu_serial_$tag.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_match -s 5 -c 1 -o gpurun_out/match_$tag python scripts/gpu_diff.py c2 60000 > gpurun_out/ncu_match_$tag.log 2>&1; tail -1 gpurun_out/ncu_match_$tag.log
