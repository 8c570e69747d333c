#!/bin/bash
# last evidence of the round: GPU tests, bench (C4) + reference arm, ncu launch list, configs C1-C3
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
tag=${1:-final2}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_$tag.log 2>&1; tail -3 gpurun_out/pytest_$tag.log
timeout 1200 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_$tag.json 2>gpurun_out/bench_$tag.err; python -c "
import json; d=json.load(open('gpurun_out/bench_$tag.json'))
print('value', round(d['value']), 'e2e', round(d['e2e']['value']), 'cpu', round(d['cpu_baseline']['value']), d['clocks'], [ (x['eviction'], round(x['value']), round(x['reference_value'])) for x in d.get('secondary',[])])"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$tag.json 2>gpurun_out/bench_ref_$tag.err; tail -c 300 gpurun_out/bench_ref_$tag.json
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv python bench.py --steps 1 --warmup 0 --no-secondary --no-traffic > gpurun_out/bench_ncu_$tag.log 2>&1; wc -l gpurun_out/launches_$tag.csv
timeout 600 python scripts/configs_report.py c1 c2 c3 > gpurun_out/configs_$tag.jsonl 2>&1; cut -c1-300 gpurun_out/configs_$tag.jsonl
