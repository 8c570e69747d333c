#!/bin/bash
# round evidence: GPU tests, bench (C4 headline) + reference arm, ncu launch list, K1/top/k_serial captures on C4, configs C1-C3
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
tag=${1:-evidence}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1800 python -m pytest tests -x -q -m gpu --durations=8 > gpurun_out/pytest_$tag.log 2>&1; tail -12 gpurun_out/pytest_$tag.log
timeout 1500 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_$tag.json 2>gpurun_out/bench_$tag.err; tail -c 1200 gpurun_out/bench_$tag.json; tail -2 gpurun_out/bench_$tag.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$tag.json 2>gpurun_out/bench_ref_$tag.err; tail -c 600 gpurun_out/bench_ref_$tag.json
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv python bench.py --steps 1 --warmup 0 --no-secondary --no-traffic > gpurun_out/bench_ncu_$tag.log 2>&1; wc -l gpurun_out/launches_$tag.csv
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_match -s 5 -c 1 -o gpurun_out/match_c4_$tag python bench.py --probe --config c4 --probe-n 100000 > gpurun_out/ncu_match_$tag.log 2>&1; tail -1 gpurun_out/ncu_match_$tag.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_top_build -s 5 -c 1 -o gpurun_out/top_c4_$tag python bench.py --probe --config c4 --probe-n 100000 > gpurun_out/ncu_top_$tag.log 2>&1; tail -1 gpurun_out/ncu_top_$tag.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_serial -s 5 -c 1 -o gpurun_out/serial_c4_$tag python bench.py --probe --config c4 --probe-n 100000 > gpurun_out/ncu_serial_$tag.log 2>&1; tail -1 gpurun_out/ncu_serial_$tag.log
timeout 600 python scripts/configs_report.py c1 c2 c3 > gpurun_out/configs_$tag.jsonl 2>&1; cut -c1-600 gpurun_out/configs_$tag.jsonl
timeout 1500 python scripts/configs_report.py c5 2>&1 | cut -c1-600 >> gpurun_out/configs_$tag.jsonl; tail -1 gpurun_out/configs_$tag.jsonl
