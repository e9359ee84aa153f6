#!/bin/bash
# k_metric variants: swap prebuilt libraries from gpurun_in/ and time cfg5 / tensor metric
for v in ${LIBS}; do
  cp gpurun_in/$v.so paper_1707_09598_b200/libsgiga.so
  for c in cfg5 cfg5_tensor cfg3; do
    timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['rooflines']
print('$v $c step', round(d['ms_per_step'],3), 'metric', round(r['metric']['ms'],3))"
  done
done
