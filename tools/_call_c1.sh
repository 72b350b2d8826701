#!/bin/bash
set -u
OUT=gpurun_out/c1; mkdir -p $OUT
for i in 1 2; do
 for v in base pre; do
  if [ $v = pre ]; then export CF_B200_LIB=build/variants/pre_ms.so; else unset CF_B200_LIB; fi
  timeout 300 python bench.py --config C1 --skip-extras --skip-schemes --skip-cpu-baseline --skip-chase > $OUT/c1_$v$i.json 2>$OUT/c1_$v$i.err
  python -c "import json;d=json.load(open('$OUT/c1_$v$i.json'));e=d['e2e'];print('$v', e['ms_per_step'], e['value'], e['frac_of_link_roofline'])"
 done
done
