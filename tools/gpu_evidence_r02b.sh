#!/bin/bash
# Round-2 evidence after the leaf-owned C4 path: GPU suite, bench lines (C2 default with
# per_config, C3, C4, C5, reference arm), launch lists, full ncu captures.  Outputs in gpurun_out/r02b/.
set -u
OUT=${OUT:-gpurun_out/r02b}; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/gputests.log 2>&1; echo "gpu tests rc=$?"; tail -2 $OUT/gputests.log
timeout 900 python bench.py > $OUT/bench_C2.json 2> $OUT/bench_C2.err; head -c 300 $OUT/bench_C2.json; echo
for CFG in C3 C4; do
  timeout 600 python bench.py --config $CFG --skip-extras > $OUT/bench_$CFG.json 2> $OUT/bench_$CFG.err; head -c 300 $OUT/bench_$CFG.json; echo
done
timeout 900 python bench.py --config C5 --steps 5 --warmup 3 --skip-chase --skip-schemes > $OUT/bench_C5.json 2> $OUT/bench_C5.err; head -c 300 $OUT/bench_C5.json; echo
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_reference_C2.json 2> $OUT/bench_reference_C2.err; head -c 300 $OUT/bench_reference_C2.json; echo
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $OUT/launches_bench_C2.csv \
  python bench.py --steps 3 --warmup 3 --skip-cpu-baseline --skip-schemes --skip-chase --skip-extras > $OUT/ncu_launch.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_resident_C4.csv \
  python tools/prof_target.py --config C4 --runs 8 --graph > $OUT/ncu_launch_c4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_scale -s 2 -c 1 -o $OUT/prof_scale_C2 -f \
  python tools/prof_target.py --config C2 --runs 3 --graph > $OUT/ncu1.log 2>&1; tail -1 $OUT/ncu1.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_" -s 4 -c 2 -o $OUT/prof_all_C4 -f \
  python tools/prof_target.py --config C4 --runs 3 --graph > $OUT/ncu2.log 2>&1; tail -1 $OUT/ncu2.log
