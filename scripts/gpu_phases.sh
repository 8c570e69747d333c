#!/bin/bash
# dev: per-phase cycles (E2_PHASES build shipped in build/) + one ncu source capture of k_serial
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
tag=${1:-x}
for c in "c2 30000" "c4 50000" "c5 8000" "c3 5000" "c1 1000"; do timeout 600 python scripts/phases.py build/libe2phases.so $c 2>&1 | tail -1; done
if [ -n "$2" ]; then
timeout 900 ncu --section SpeedOfLight --section WarpStateStats --section SourceCounters --section InstructionStats --clock-control none --import-source on -k regex:k_serial -s 0 -c 1 -o gpurun_out/serial_$tag python scripts/gpu_diff.py $2 $3 > gpurun_out/ncu_serial_$tag.log 2>&1; tail -2 gpurun_out/ncu_serial_$tag.log
fi
