#!/bin/bash
# dev: one ncu --set full capture of k_serial on C4 (a 16k-request batch) + source-level summary
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
tag=${1:-x}
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_serial -s 5 -c 1 -o gpurun_out/serial_c4_$tag python bench.py --probe --config c4 --probe-n 100000 > gpurun_out/ncu_serial_$tag.log 2>&1; tail -2 gpurun_out/ncu_serial_$tag.log
python scripts/ncu_lines.py gpurun_out/serial_c4_$tag.ncu-rep 60 > gpurun_out/serial_lines_$tag.txt 2>&1; head -80 gpurun_out/serial_lines_$tag.txt
