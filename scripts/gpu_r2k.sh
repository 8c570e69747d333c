#!/bin/bash
# dev: parity subset + phases + decisions/s after the serial-path changes
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_parity.py tests/test_deep_paths.py tests/test_golden.py tests/test_fuzz.py tests/test_replay_errors.py tests/test_reference_unit.py -x -q -m gpu -k "not c5" 2>&1 | tail -3
for c in c4:100000 c2:30000 c1:1000; do timeout 600 python scripts/phases.py build/libe2phases.so ${c%%:*} ${c##*:} 2>&1 | tail -1; done
timeout 900 python scripts/ab_time.py paper_2407_00023_b200/libe2sched.so c4 100000 3
timeout 900 python scripts/ab_time.py paper_2407_00023_b200/libe2sched.so c2 100000 3
timeout 900 python scripts/ab_time.py paper_2407_00023_b200/libe2sched.so c1 1000 5
