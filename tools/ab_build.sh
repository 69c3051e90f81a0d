#!/bin/bash
# Build a variant of libhpz.so into $1/libhpz.so with extra nvcc flags ($2...), for A/B runs
# (HPZ_LIB=$1/libhpz.so python bench.py ...).  Same sources and flags as build.py.
set -e
OUT=$1; shift
mkdir -p "$OUT"
cd "$(dirname "$0")/.."
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --shared -Xcompiler -fPIC \
  -Xcompiler -fvisibility=hidden -I include -Xptxas -O3 -o "$OUT/libhpz.so" \
  paper_2407_01614_b200/csrc/hpz_kernels.cu paper_2407_01614_b200/csrc/hpz_tma.cu paper_2407_01614_b200/csrc/hpz_runtime.cpp \
  -Xcompiler -Wall "$@"
