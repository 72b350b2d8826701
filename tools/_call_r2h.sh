#!/bin/bash
set -u
OUT=gpurun_out/r2h; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/gputests.log 2>&1; echo "gpu tests rc=$?"; grep -E "passed|failed|FAILED|Error" $OUT/gputests.log | tail -15
