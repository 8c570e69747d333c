#!/bin/bash
# dev: per-call session checks: per-call GPU tests, per-call latency with and without the session
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
tag=${1:-x}
timeout 900 python -m pytest tests -x -q -m gpu -k "fuzz or reference_unit or dropin or snapshot or abi" > gpurun_out/pytest_$tag.log 2>&1; tail -3 gpurun_out/pytest_$tag.log
timeout 300 python scripts/percall.py 2000
E2_NO_SESSION=1 timeout 300 python scripts/percall.py 2000
make -s -C oracle _ref/drop_in_b200 2>/dev/null; ls oracle/_ref/drop_in_b200 && timeout 300 oracle/_ref/drop_in_b200 3000 && E2_NO_SESSION=1 timeout 300 oracle/_ref/drop_in_b200 3000
