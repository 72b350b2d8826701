#!/bin/bash
# Build experimental variants of the library (design experiments only): build/variants/<name>.so
set -e
mkdir -p build/variants
v() { name=$1; shift; mkdir -p build/variants/$name; \
  for f in cf_kernels.cu cf_runtime.cpp cf_tree.cpp cf_ops.cpp cf_window.cpp; do \
    x=""; [[ $f == *.cpp ]] && x="-x cu"; \
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -ccbin /usr/bin/g++ -Xcompiler -fPIC,-fopenmp -Iinclude $x "$@" -c paper_1906_01128_b200/csrc/$f -o build/variants/$name/${f%.*}.o & done; wait; \
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -ccbin /usr/bin/g++ -Xcompiler -fopenmp -o build/variants/$name.so build/variants/$name/*.o -lgomp; }
v base
v minb8 -DCF_SCALE_MINB=8
v g32 -DCF_GROUP_KB=32
v g32u8 -DCF_GROUP_KB=32 -DCF_GROUP_U=8
v g32minb8 -DCF_GROUP_KB=32 -DCF_SCALE_MINB=8
v g8 -DCF_GROUP_KB=8 -DCF_GROUP_U=2
