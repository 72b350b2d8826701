#!/bin/bash
# Runs on the GPU box (under gpurun): bench line, kernel launch list, one full ncu capture of
# the leaf kernel and of the relocation kernel.  Outputs land in gpurun_out/.
set -u
OUT=gpurun_out
mkdir -p $OUT
CFG=${CFG:-C2}
timeout 600 python bench.py --config $CFG > $OUT/bench_$CFG.json 2> $OUT/bench_$CFG.err
tail -c 3000 $OUT/bench_$CFG.err
cat $OUT/bench_$CFG.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $OUT/launches_$CFG.csv python bench.py --config $CFG --steps 3 --warmup 3 --skip-cpu-baseline \
  > $OUT/ncu_launch_run.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_scale -s 6 -c 2 \
  -o $OUT/prof_scale_$CFG -f python bench.py --config $CFG --steps 3 --warmup 3 --skip-cpu-baseline --skip-chase \
  > $OUT/ncu_full_run.log 2>&1
tail -5 $OUT/ncu_full_run.log
