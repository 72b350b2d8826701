#!/bin/bash
# Round-2 re-entry check: GPU test suite, smoke, default bench line, reference arm.
set -u
OUT=gpurun_out/v1; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/gputests.log 2>&1; echo "gpu tests rc=$?"; tail -3 $OUT/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; head -c 400 $OUT/bench.json; echo
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "ref rc=$?"; head -c 300 $OUT/bench_ref.json; echo
