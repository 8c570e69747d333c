#!/bin/bash
# dev: GPU tests + per-phase cycles + quick bench line
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
tag=${1:-x}
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_$tag.log 2>&1; tail -3 gpurun_out/pytest_$tag.log
bash scripts/gpu_phq.sh $tag
