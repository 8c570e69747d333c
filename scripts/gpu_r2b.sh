#!/bin/bash
# round 2: bench line (C4 headline) + reference arm + one source-level ncu capture of k_serial on C4
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
tag=${1:-r2b}
timeout 1500 python bench.py --steps ${STEPS:-3} --warmup 2 > gpurun_out/bench_$tag.json 2>gpurun_out/bench_$tag.err; tail -c 2500 gpurun_out/bench_$tag.json; tail -3 gpurun_out/bench_$tag.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$tag.json 2>&1; tail -c 600 gpurun_out/bench_ref_$tag.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_serial -s 5 -c 1 -o gpurun_out/serial_c4_$tag python bench.py --probe --config c4 --probe-n 100000 > gpurun_out/ncu_serial_$tag.log 2>&1; tail -2 gpurun_out/ncu_serial_$tag.log
