#!/bin/bash
# round 2: GPU tests (sharded device path, streamed C5, larger parity sizes, fuzz 1000) + sanitizers
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_r2f.log 2>&1; tail -5 gpurun_out/pytest_r2f.log
for tool in racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize.py c2 5000 > gpurun_out/sanitize_${tool}_c2.log 2>&1; echo "$tool rc=$?"; tail -4 gpurun_out/sanitize_${tool}_c2.log
done
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python scripts/sanitize.py c4 5000 > gpurun_out/sanitize_memcheck_c4.log 2>&1; echo "memcheck rc=$?"; tail -4 gpurun_out/sanitize_memcheck_c4.log
