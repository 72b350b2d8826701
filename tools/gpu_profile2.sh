#!/bin/bash
# Resident-step launch lists and full ncu captures (k_scale for C2; all kernels for C4).
set -u
OUT=gpurun_out; mkdir -p $OUT
for CFG in C1 C4; do
  timeout 600 python bench.py --config $CFG --skip-cpu-baseline > $OUT/bench_$CFG.json 2> $OUT/bench_$CFG.err; cat $OUT/bench_$CFG.json; tail -3 $OUT/bench_$CFG.err
done
for CFG in C2 C4; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_resident_$CFG.csv \
    python tools/prof_target.py --config $CFG --runs 3 > /dev/null 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_scale -s 2 -c 1 -o $OUT/prof_scale_C2 -f \
  python tools/prof_target.py --config C2 --runs 3 > $OUT/ncu1.log 2>&1; tail -2 $OUT/ncu1.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_" -s 8 -c 4 -o $OUT/prof_all_C4 -f \
  python tools/prof_target.py --config C4 --runs 3 > $OUT/ncu2.log 2>&1; tail -2 $OUT/ncu2.log
