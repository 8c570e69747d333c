#!/bin/bash
# dev: instrumented variant build: build/lib$1.so with extra -D flags ($2...)
cd "$(dirname "$0")/.."
mkdir -p build
name=$1; shift
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared "$@" \
  -Iinclude -o build/lib$name.so paper_2407_00023_b200/csrc/e2_lib.cu paper_2407_00023_b200/csrc/workload_gen.cpp paper_2407_00023_b200/csrc/corpus.cpp
