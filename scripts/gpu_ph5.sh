#!/bin/bash
cd $GRAFT_REPO_ROOT
for c in c4:100000; do timeout 600 python scripts/phases.py build/libe2phases.so ${c%%:*} ${c##*:} 2>&1 | tail -1; done
