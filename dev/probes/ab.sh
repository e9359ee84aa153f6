#!/bin/bash
# A/B of prebuilt libraries (gpurun_in/<name>.so) on one box: LIBS="old new" CFGS="cfg5"
for rep in 1 2; do
for v in ${LIBS}; do
  cp gpurun_in/$v.so paper_1707_09598_b200/libsgiga.so
  for c in ${CFGS:-cfg5}; do
    timeout 300 python bench.py --config $c --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['rooflines']
print('$v $c', round(d['ms_per_step'],3), {k:round(v['ms'],3) for k,v in r.items() if v['ms']>0.05}, d.get('clocks',{}).get('sm_mhz'))"
  done
done
done
