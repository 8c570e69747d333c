#!/bin/bash
# dev: per-phase cycles (instrumented build) + quick bench line
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
tag=${1:-x}
for c in ${PH_CONFIGS:-c2:30000 c5:8000}; do timeout 600 python scripts/phases.py ${PH_LIB:-build/libe2phases.so} ${c%%:*} ${c##*:} 2>&1 | tail -1; done
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_$tag.json 2>gpurun_out/bench_$tag.err; python -c "
import json; d=json.load(open('gpurun_out/bench_$tag.json'))
print('value', round(d['value']), 'e2e', round(d['e2e']['value']), 'serial ms/step', round(d['kernel_ms_per_step']['serial_commit'],1), 'match frac', round(d['roofline']['frac'],3), 'match ms', d['roofline']['avg_launch_ms'], 'cpu', round(d['cpu_baseline']['value']))"; tail -2 gpurun_out/bench_$tag.err
