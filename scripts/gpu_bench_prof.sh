#!/bin/bash
# dev: quick perf check of the serial kernel (tests optional via $1=tests)
cd $GRAFT_REPO_ROOT
if [ "$1" == "tests" ]; then timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3; fi
timeout 600 python bench.py --steps 3 --warmup 1 > gpurun_out/bench_$2.json 2>gpurun_out/bench_$2.err; python -c "
import json; d=json.load(open('gpurun_out/bench_$2.json'))
print('value', round(d['value']), 'e2e', round(d['e2e']['value']), 'serial ms/step', round(d['kernel_ms_per_step']['serial_commit'],1), 'match frac', round(d['roofline']['frac'],3), 'cpu', round(d['cpu_baseline']['value']))"; tail -2 gpurun_out/bench_$2.err
timeout 600 ncu --section SpeedOfLight --section WarpStateStats --section SourceCounters --section InstructionStats --clock-control none --import-source on -k regex:k_serial -s 0 -c 1 -o gpurun_out/serial_$2 python scripts/gpu_diff.py c2 20000 > gpurun_out/ncu_serial_$2.log 2>&1; tail -1 gpurun_out/ncu_serial_$2.log
