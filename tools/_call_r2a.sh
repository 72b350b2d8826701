#!/bin/bash
# uniform memory-parallel resolver + PDL + reloc-first detach: parity, then A/B timing
set -u
OUT=gpurun_out/r2a; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_uniform_resolve.py tests/test_gpu_fullsize.py tests/test_gpu_faults.py tests/test_gpu_parity.py -x -q -p no:cacheprovider > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -3 $OUT/tests.log
timeout 900 python tools/r2_env_ab.py C4 C2 -- base CF_NO_PDL=1 CF_UNI_U=4 CF_UNI_U=2 CF_NO_UNI=1 CF_NO_UNI=1,CF_NO_PDL=1 > $OUT/ab.log 2>&1; cat $OUT/ab.log
