#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python scripts/ab_time.py build/libbase.so,build/libpfl.so c4 100000 3
E2_NO_PREFETCH=1 timeout 900 python scripts/ab_time.py build/libpfl.so c4 100000 3
timeout 900 python scripts/ab_time.py build/libbase.so,build/libpfl.so c2 100000 3
E2_NO_PREFETCH=1 timeout 900 python scripts/ab_time.py build/libpfl.so c2 100000 3
