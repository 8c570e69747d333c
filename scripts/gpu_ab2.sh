#!/bin/bash
# dev: A/B of library builds on one box: C4/C2/C1 kernel-time decisions/s + C5 streamed
cd $GRAFT_REPO_ROOT
L=${AB_LIBS:-paper_2407_00023_b200/libe2sched.so,build/libpf.so}
for c in ${AB_CONFIGS:-c4:100000 c2:100000 c1:1000}; do timeout 600 python scripts/ab_time.py $L ${c%%:*} ${c##*:} 2>&1 | tail -8; done
timeout 900 python scripts/ab_c5.py $L ${C5N:-196608} 2>&1 | tail -8
