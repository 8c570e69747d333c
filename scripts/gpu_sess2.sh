#!/bin/bash
# dev: per-call session: GPU tests (per-call ones first) + latency
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
tag=${1:-x}
E2_SESSION_DEBUG=1 timeout 120 python scripts/percall.py 2000
timeout 120 oracle/_ref/drop_in_b200 3000
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_$tag.log 2>&1; tail -3 gpurun_out/pytest_$tag.log
