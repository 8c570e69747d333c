#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python scripts/ab_k1.py build/libcur.so,build/libk1b6.so,build/libk1b8.so c4 100000
timeout 900 python scripts/ab_k1.py build/libcur.so,build/libk1b6.so,build/libk1b8.so c2 100000
timeout 300 python scripts/percall.py 2000
timeout 300 python -m pytest tests/test_dropin_cpp.py -q -m gpu -s 2>&1 | grep -E "per-call|passed|failed"
timeout 900 python scripts/c5_rate.py 200000
