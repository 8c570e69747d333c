#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -q -m gpu -k "not c5-100000" 2>&1 | tail -2
timeout 900 python scripts/ab_time.py build/libprecache.so,paper_2407_00023_b200/libe2sched.so c4 100000 3
timeout 900 python scripts/ab_time.py build/libprecache.so,paper_2407_00023_b200/libe2sched.so c2 100000 3
timeout 900 python scripts/c5_rate.py 131072
