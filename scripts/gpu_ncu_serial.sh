#!/bin/bash
# dev: one ncu --set full capture of k_serial (first C2 batch after the ramp) + source-level summary
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
tag=${1:-x}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_serial -s ${2:-8} -c 1 -o gpurun_out/serial_$tag python scripts/gpu_diff.py c2 60000 > gpurun_out/ncu_serial_$tag.log 2>&1; tail -2 gpurun_out/ncu_serial_$tag.log
