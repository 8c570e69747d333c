#!/bin/bash
# dev: GPU parity subset + A/B of a candidate build against the previous one (build/libprev.so)
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_parity.py tests/test_fuzz.py tests/test_deep_paths.py tests/test_reference_unit.py tests/test_replay_errors.py -q -m gpu -k "not c5-100000 and not c4-None" 2>&1 | tail -2
for c in c4:100000:3 c2:100000:3 c1:1000:5; do IFS=: read n m r <<< "$c"; timeout 900 python scripts/ab_time.py build/libprev.so,paper_2407_00023_b200/libe2sched.so $n $m $r; done
