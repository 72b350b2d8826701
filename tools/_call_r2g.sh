#!/bin/bash
set -u
OUT=gpurun_out/r2g; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/gputests.log 2>&1; echo "gpu tests rc=$?"; tail -30 $OUT/gputests.log | grep -v "^\.\.\.\."
timeout 600 python tools/c4_tables_probe.py C4 C2 > $OUT/tab.log 2>&1; cat $OUT/tab.log
CF_NO_LEAF_OWN=1 timeout 600 python tools/c4_tables_probe.py C4 > $OUT/tab_noown.log 2>&1; cat $OUT/tab_noown.log
timeout 600 python tools/r2_env_ab.py C4 C2 > $OUT/ab.log 2>&1; cat $OUT/ab.log
