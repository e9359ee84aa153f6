#!/bin/bash
# cluster-assembly probe: parity subset, then assembly times of the variants
python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_r2.py -m gpu -q -p no:cacheprovider -x \
  -k "cfg5 or cfg2 or tensor or permutation or assembl or tma" 2>&1 | tail -4
for v in "" "SGIGA_ASM_CL_NGB3=1" "SGIGA_NO_ASM_CLUSTER=1"; do
  for c in ${CFGS:-cfg5 cfg2}; do
    env $v python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['rooflines']
print('$v', d['config']['workload'], round(d['ms_per_step'],3), {k:(round(v['ms'],3), round(v.get('frac',0),3)) for k,v in r.items()})"
  done
done
for v in "" "SGIGA_ASM_CL_NGB3=1"; do
  env $v SGIGA_ASM_PROFILE=1 python - <<'PY' 2>&1 | grep asm-profile | tail -1
import sys; sys.path.insert(0, '.')
from paper_1707_09598_b200 import configs
from paper_1707_09598_b200.pipeline import Batch
from paper_1707_09598_b200.scheduler import make_spec
cfg = configs.get_config('cfg5')
b = Batch(make_spec(tuple(cfg.plan.terms), cfg.problem, cfg.quad_points))
for _ in range(2): b.assemble()
b.close()
PY
done
