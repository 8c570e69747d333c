#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python scripts/phases_c5.py build/libe2phases.so 262144 2>&1 | tail -5
