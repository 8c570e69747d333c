#!/bin/bash
# dev: first device run
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 compute-sanitizer --tool memcheck --error-exitcode 9 python scripts/gpu_diff.py c1 300 - 32 2>&1 | tail -15
timeout 300 python scripts/gpu_diff.py c1 1000 2>&1 | tail -5
timeout 300 python scripts/gpu_diff.py c1 1000 - 64 2>&1 | tail -5
timeout 600 python scripts/gpu_diff.py c2 20000 2>&1 | tail -5
timeout 900 python scripts/gpu_diff.py c2 100000 2>&1 | tail -5
