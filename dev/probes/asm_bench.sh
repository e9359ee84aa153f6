#!/bin/bash
# assembly / phase timings of replicated batches: asm_bench.sh cfg3:1024 cfg1:1024 ...
for a in "$@"; do
  c=${a%%:*}; r=${a##*:}
  python bench.py --config $c --replicas $r --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['rooflines']
print(d['config']['workload'], 'x$r', round(d['ms_per_step'],3), {k:(round(v['ms'],3), round(v.get('frac',0),3)) for k,v in r.items()})"
done
