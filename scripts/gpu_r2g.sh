#!/bin/bash
# round 2: staged K1 + barrier fixes: GPU tests, sanitizers, C4 bench line
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -x -q -m gpu --durations=12 > gpurun_out/pytest_r2g.log 2>&1; tail -22 gpurun_out/pytest_r2g.log
for tool in synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 200 python scripts/sanitize.py c2 5000 > gpurun_out/sanitize_${tool}_c2_r2g.log 2>&1; echo "$tool rc=$?"; tail -3 gpurun_out/sanitize_${tool}_c2_r2g.log
done
timeout 1500 python bench.py --steps 3 --warmup 3 --no-secondary > gpurun_out/bench_r2g.json 2>gpurun_out/bench_r2g.err; python -c "
import json; d=json.loads(open('gpurun_out/bench_r2g.json').read().strip().splitlines()[-1])
print({k: d[k] for k in ('value','ms_per_step')}, d['e2e']['value'], d['roofline_k1'], d['kernel_ms_per_step'], d['cpu_baseline']['value'])"; tail -2 gpurun_out/bench_r2g.err
