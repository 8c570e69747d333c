#!/bin/bash
# dev: phases of variant libs: $1 tag, $2.. lib names (build/lib<name>.so); configs from PH_CONFIGS
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
tag=$1; shift
for L in "$@"; do
  echo "== $L"
  for c in ${PH_CONFIGS:-c2:100000}; do timeout 600 python scripts/phases.py build/lib$L.so ${c%%:*} ${c##*:} 2>&1 | tail -1; done
done
