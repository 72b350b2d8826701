#!/bin/bash
# Round-2 evidence after multi-step leaf-owned windows: bench lines C2 (default) and C4, the C4
# e2e window's launch list.  Outputs in gpurun_out/r02c/.
set -u
OUT=gpurun_out/r02c; mkdir -p $OUT
timeout 900 python bench.py > $OUT/bench_C2.json 2> $OUT/bench_C2.err; head -c 300 $OUT/bench_C2.json; echo
timeout 600 python bench.py --config C4 --skip-extras > $OUT/bench_C4.json 2> $OUT/bench_C4.err; head -c 300 $OUT/bench_C4.json; echo
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $OUT/launches_e2e_C4.csv \
  python tools/prof_target.py --config C4 --runs 2 --full > $OUT/ncu_e2e_c4.log 2>&1; tail -1 $OUT/ncu_e2e_c4.log
