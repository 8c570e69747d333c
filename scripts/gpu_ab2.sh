#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_parity.py tests/test_deep_paths.py tests/test_replay_errors.py tests/test_golden.py -x -q -m gpu -k "not c5" 2>&1 | tail -2
timeout 900 python scripts/ab_time.py build/libpre.so,build/libpfc2.so c4 100000 3
timeout 900 python scripts/ab_time.py build/libpre.so,build/libpfc2.so c2 100000 3
timeout 900 python scripts/ab_time.py build/libpre.so,build/libpfc2.so c1 1000 5
timeout 900 python scripts/ab_time.py build/libpre.so,build/libpfc2.so c3 10000 3
