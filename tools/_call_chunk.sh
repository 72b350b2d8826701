#!/bin/bash
set -u
OUT=gpurun_out/chunk; mkdir -p $OUT
for i in 1 2; do
 for mb in 32 64 128 16; do
  timeout 300 python bench.py --config C2 --skip-extras --skip-schemes --skip-cpu-baseline --skip-chase --chunk-mb $mb > $OUT/c2_${mb}_${i}.json 2>/dev/null
  python -c "import json;d=json.load(open('$OUT/c2_${mb}_${i}.json'));e=d['e2e'];print('$mb', e['ms_per_step'], e['value'], e['frac_of_link_roofline'], e['host_link_gbs']['bidir'], e['pipeline_link_gbs']['bidir'])"
 done
done
