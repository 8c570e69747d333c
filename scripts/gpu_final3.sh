#!/bin/bash
# dev: A/B of the path-scratch size, then GPU tests + bench on the product
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
tag=${1:-final3}
AB_LIBS=paper_2407_00023_b200/libe2sched.so,build/libl1p256.so AB_CONFIGS="c4:100000 c2:100000" C5N=65536 bash scripts/gpu_ab2.sh
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_$tag.log 2>&1; tail -3 gpurun_out/pytest_$tag.log
timeout 1200 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_$tag.json 2>gpurun_out/bench_$tag.err; python -c "
import json; d=json.load(open('gpurun_out/bench_$tag.json'))
print('value', round(d['value']), 'e2e', round(d['e2e']['value']), 'cpu', round(d['cpu_baseline']['value']), d['clocks'], [ (x['eviction'], round(x['value']), round(x['reference_value'])) for x in d.get('secondary',[])])"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$tag.json 2>gpurun_out/bench_ref_$tag.err; tail -c 300 gpurun_out/bench_ref_$tag.json
timeout 600 python scripts/configs_report.py c1 c2 c3 > gpurun_out/configs_$tag.jsonl 2>&1; cut -c1-250 gpurun_out/configs_$tag.jsonl
python -c "import __graft_entry__ as g; g.smoke()"
