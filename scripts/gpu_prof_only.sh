#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 ncu --section SpeedOfLight --section WarpStateStats --section SourceCounters --section InstructionStats --clock-control none --import-source on -k regex:k_serial -s 0 -c 1 -o gpurun_out/serial_$1 python scripts/gpu_diff.py $2 $3 > gpurun_out/ncu_serial_$1.log 2>&1; tail -1 gpurun_out/ncu_serial_$1.log
