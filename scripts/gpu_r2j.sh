#!/bin/bash
# dev: phases on C4/C2 (inline children build), K1 tile A/B, total decisions/s A/B
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in c4:100000 c2:30000; do timeout 600 python scripts/phases.py build/libe2phases.so ${c%%:*} ${c##*:} 2>&1 | tail -1; done
timeout 900 python scripts/ab_k1.py paper_2407_00023_b200/libe2sched.so,build/libtile1.so,build/libtile2.so c4 100000
E2_NO_TOP=1 timeout 600 python scripts/ab_k1.py build/libtile1.so c4 100000
timeout 900 python scripts/ab_k1.py paper_2407_00023_b200/libe2sched.so,build/libtile1.so c2 100000
E2_NO_TOP=1 timeout 600 python scripts/ab_k1.py build/libtile1.so c2 100000
