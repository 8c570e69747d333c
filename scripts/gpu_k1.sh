#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_parity.py tests/test_deep_paths.py tests/test_golden.py tests/test_reference_unit.py -x -q -m gpu -k "not c5" 2>&1 | tail -2
timeout 900 python scripts/ab_k1.py paper_2407_00023_b200/libe2sched.so,build/k1seq.so c4 100000 2>&1 | tail -2
timeout 900 python scripts/ab_k1.py paper_2407_00023_b200/libe2sched.so,build/libk1seq.so c4 100000
timeout 900 python scripts/ab_k1.py paper_2407_00023_b200/libe2sched.so,build/libk1seq.so c2 100000
timeout 900 python scripts/ab_k1.py paper_2407_00023_b200/libe2sched.so,build/libk1seq.so c3 10000
