#!/bin/sh
# UVM prefetch-pipelined window (CF_WIN_UVM) step size vs window time, C2 (design experiment)
for mb in 32 128 256 1024; do
  echo "chunk ${mb} MiB"; CF_UVM_CHUNK_MB=$mb python tools/time_schemes.py C2 uvm_prefetch 2>&1 | tail -2
done
