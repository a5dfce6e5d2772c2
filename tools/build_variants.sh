#!/bin/bash
# Build A/B variants of libdtb_b200.so into ab/ (fp64 only is fine for timing).
set -e
cd "$(dirname "$0")/.."
mkdir -p ab
build() {  # name, defines...
  local name=$1; shift
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 \
    -Xcompiler -fPIC -shared "$@" paper_2306_03336_b200/csrc/dtb_kernels.cu \
    paper_2306_03336_b200/csrc/dtb_plan.cpp -o ab/lib_$name.so &
}
build "$@"
wait
