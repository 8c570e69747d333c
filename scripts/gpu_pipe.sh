#!/bin/bash
# dev: pipelined vs single-warp replay: tests (default), phases for both, bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
tag=${1:-x}
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_$tag.log 2>&1; tail -3 gpurun_out/pytest_$tag.log
for np in 0 1; do
  echo "== E2_NO_PIPE=$np"
  for c in ${PH_CONFIGS:-c2:100000}; do E2_NO_PIPE=$np timeout 600 python scripts/phases.py build/libe2phases.so ${c%%:*} ${c##*:} 2>&1 | tail -1; done
done
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_$tag.json 2>gpurun_out/bench_$tag.err; python -c "
import json; d=json.load(open('gpurun_out/bench_$tag.json'))
print('value', round(d['value']), 'e2e', round(d['e2e']['value']), 'serial ms/step', round(d['kernel_ms_per_step']['serial_commit'],1), 'match frac', round(d['roofline']['frac'],3), 'cpu', round(d['cpu_baseline']['value']))"; tail -2 gpurun_out/bench_$tag.err
