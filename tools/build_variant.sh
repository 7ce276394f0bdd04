#!/bin/bash
# build libdvm.so with extra nvcc defines into tools/ab/libdvm_$1.so (A/B timing only)
NAME=$1; shift
mkdir -p tools/ab
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC \
  -Xcompiler -fvisibility=hidden -shared -fmad=true "$@" -I include paper_1201_3986_b200/csrc/*.cu -o tools/ab/libdvm_$NAME.so
