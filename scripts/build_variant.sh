#!/bin/bash
# build libdlic.so with extra -D flags into OUT: scripts/build_variant.sh OUT.so -DFOO=1 ...
OUT=$1; shift
cd "$(dirname "$0")/../paper_2207_05152_b200/csrc"
nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC -shared "$@" -o "$OUT" dlic_kernels.cu dlic_api.cu
