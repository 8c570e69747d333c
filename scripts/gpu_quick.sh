#!/bin/bash
# dev: GPU tests + one bench line (+ optional ncu of one kernel: $2 = kernel regex)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
tag=${1:-x}
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_$tag.log 2>&1; tail -3 gpurun_out/pytest_$tag.log
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_$tag.json 2>gpurun_out/bench_$tag.err; python -c "
import json; d=json.load(open('gpurun_out/bench_$tag.json'))
print('value', round(d['value']), 'e2e', round(d['e2e']['value']), 'serial ms/step', round(d['kernel_ms_per_step']['serial_commit'],1), 'match frac', round(d['roofline']['frac'],3), 'match ms', d['roofline']['avg_launch_ms'], 'cpu', round(d['cpu_baseline']['value']))"; tail -2 gpurun_out/bench_$tag.err
if [ -n "$2" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s ${3:-1} -c 1 -o gpurun_out/${2}_$tag python scripts/gpu_diff.py c2 40000 > gpurun_out/ncu_${2}_$tag.log 2>&1; tail -2 gpurun_out/ncu_${2}_$tag.log
fi
