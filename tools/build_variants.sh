#!/bin/bash
# Build experimental variants of the library (design experiments only): build/variants/<name>.so
set -e
mkdir -p build/variants
v() { name=$1; shift; mkdir -p build/variants/$name; \
  for f in cf_kernels.cu cf_runtime.cpp cf_tree.cpp cf_ops.cpp cf_window.cpp cf_selective.cpp; do \
    x=""; [[ $f == *.cpp ]] && x="-x cu"; \
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -ccbin /usr/bin/g++ -Xcompiler -fPIC,-fopenmp -Iinclude $x "$@" -c paper_1906_01128_b200/csrc/$f -o build/variants/$name/${f%.*}.o & done; wait; \
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -ccbin /usr/bin/g++ -Xcompiler -fopenmp -o build/variants/$name.so build/variants/$name/*.o -lgomp; }
if [ $# -gt 0 ]; then v "$@"; exit 0; fi
v blockgrp -DCF_GROUP_WARP=0
v warp8 -DCF_GROUP_WARP=1 -DCF_SCALE_MINB=8
v warp6 -DCF_GROUP_WARP=1 -DCF_SCALE_MINB=6
v warp4 -DCF_GROUP_WARP=1 -DCF_SCALE_MINB=4
