#!/bin/bash
# dev: the reference harness on the drop-in with stderr shown; per-call latency with/without the session
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/e2e_dbg
#timeout 120 oracle/_ref/e2e_dropin_b200 gpurun_out/e2e_dbg 2>&1 | tail -5
E2_SESSION_DEBUG=1 timeout 120 python scripts/percall.py 2000
E2_NO_SESSION=1 timeout 120 python scripts/percall.py 2000
timeout 120 oracle/_ref/drop_in_b200 3000 && E2_NO_SESSION=1 timeout 120 oracle/_ref/drop_in_b200 3000
