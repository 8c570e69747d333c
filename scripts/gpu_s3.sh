#!/bin/bash
# dev: GPU tests, one bench line, per-phase cycles on C4/C1 (instrumented build)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
tag=${1:-x}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
if [ -z "$NO_TESTS" ]; then timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_$tag.log 2>&1; tail -3 gpurun_out/pytest_$tag.log; fi
timeout 900 python bench.py --steps 3 --warmup 3 --no-secondary > gpurun_out/bench_$tag.json 2>gpurun_out/bench_$tag.err; python -c "
import json; d=json.load(open('gpurun_out/bench_$tag.json'))
print('value', round(d['value']), 'e2e', round(d['e2e']['value']), 'ms/step', round(d['ms_per_step'],1), 'cpu', round(d['cpu_baseline']['value']), d.get('clocks'))"; tail -2 gpurun_out/bench_$tag.err
for c in ${PH_CONFIGS:-c4:100000 c1:1000}; do timeout 600 python scripts/phases.py ${PH_LIB:-build/libe2phases.so} ${c%%:*} ${c##*:} 2>&1 | tail -1; done
for c in ${AB_CONFIGS:-c4:100000 c2:100000 c1:1000}; do timeout 600 python scripts/ab_time.py ${AB_LIBS:-paper_2407_00023_b200/libe2sched.so} ${c%%:*} ${c##*:} 2>&1 | tail -3; done
