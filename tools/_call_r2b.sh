#!/bin/bash
set -u
OUT=gpurun_out/r2b; mkdir -p $OUT
timeout 900 python tools/r2_env_ab.py C4 C2 -- base CF_RELOC_FIRST=1 CF_NO_PDL=1 > $OUT/ab.log 2>&1; cat $OUT/ab.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 60 --csv --log-file $OUT/launches_C4_graph.csv \
  python tools/prof_target.py --config C4 --runs 12 --graph > $OUT/ncu_c4.log 2>&1; tail -2 $OUT/ncu_c4.log
python tools/launch_summary.py $OUT/launches_C4_graph.csv $OUT/launches_C4_graph.md "C4 resident graph steps (warm cache)" 2>&1 | tail -8; grep -o "\"k_[a-z_]*[^\"]*\",\"[^\"]*\",\"[^\"]*\",\"[0-9.,]*\"" $OUT/launches_C4_graph.csv | tail -6
timeout 600 python -m pytest tests/test_gpu_uniform_resolve.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider -k "uniform or C4 or C2 or many" > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -2 $OUT/tests.log
