#!/bin/bash
# dev: instrumented build (per-phase clock64 totals) -> build/libe2phases.so
cd "$(dirname "$0")/.."
mkdir -p build
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -DE2_PHASES \
  -Iinclude -o build/libe2phases.so paper_2407_00023_b200/csrc/e2_lib.cu paper_2407_00023_b200/csrc/workload_gen.cpp paper_2407_00023_b200/csrc/corpus.cpp
