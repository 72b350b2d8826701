#!/bin/bash
set -u
OUT=gpurun_out/r2f; mkdir -p $OUT
V=build/variants
timeout 1200 python tools/r2_env_ab.py C4 C2 -- CF_NO_LEAF_OWN=1 CF_NO_LEAF_OWN=1,CF_B200_LIB=$V/grp_m4_u8.so CF_NO_LEAF_OWN=1,CF_B200_LIB=$V/grp_m4_u4.so CF_NO_LEAF_OWN=1,CF_B200_LIB=$V/grp_m5_u4.so CF_NO_LEAF_OWN=1,CF_B200_LIB=$V/grp_m5_u8.so > $OUT/ab.log 2>&1; cat $OUT/ab.log
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -x -q -p no:cacheprovider -k sanitizer > $OUT/san.log 2>&1; echo "san rc=$?"; tail -3 $OUT/san.log
