#!/bin/bash
# round evidence (final): GPU tests, bench (C4 headline) + reference arm, ncu launch list,
# K1 capture, configs report C1-C3 + C5, per-call session latency
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
tag=${1:-final}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest tests -x -q -m gpu --durations=8 > gpurun_out/pytest_$tag.log 2>&1; tail -12 gpurun_out/pytest_$tag.log
timeout 1200 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_$tag.json 2>gpurun_out/bench_$tag.err; tail -c 1500 gpurun_out/bench_$tag.json; tail -2 gpurun_out/bench_$tag.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$tag.json 2>gpurun_out/bench_ref_$tag.err; tail -c 600 gpurun_out/bench_ref_$tag.json
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv python bench.py --steps 1 --warmup 0 --no-secondary --no-traffic > gpurun_out/bench_ncu_$tag.log 2>&1; wc -l gpurun_out/launches_$tag.csv
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_match -s 5 -c 1 -o gpurun_out/match_c4_$tag python bench.py --probe --config c4 --probe-n 100000 > gpurun_out/ncu_match_$tag.log 2>&1; tail -1 gpurun_out/ncu_match_$tag.log
timeout 600 python scripts/configs_report.py c1 c2 c3 > gpurun_out/configs_$tag.jsonl 2>&1; cut -c1-600 gpurun_out/configs_$tag.jsonl
timeout 1500 python scripts/configs_report.py c5 2>&1 | cut -c1-600 >> gpurun_out/configs_$tag.jsonl; tail -1 gpurun_out/configs_$tag.jsonl
E2_SESSION_DEBUG=1 timeout 120 python scripts/percall.py 2000 > gpurun_out/percall_$tag.log 2>&1; E2_NO_SESSION=1 timeout 120 python scripts/percall.py 2000 >> gpurun_out/percall_$tag.log 2>&1; cat gpurun_out/percall_$tag.log
timeout 120 oracle/_ref/drop_in_b200 3000 | tee -a gpurun_out/percall_$tag.log
timeout 900 python scripts/ab_c5.py paper_2407_00023_b200/libe2sched.so 262144 2>&1 | tail -1 | tee gpurun_out/c5_stream_$tag.log
