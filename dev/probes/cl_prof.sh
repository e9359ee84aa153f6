#!/bin/bash
# stage profile + assembly time of the 3-D assembly variants on cfg5 (block 0)
for v in ${VARIANTS:-"SGIGA_NO_ASM_CLUSTER=1" "SGIGA_ASM_CL_NGB3=1" "SGIGA_ASM_CL_NGB3=0"}; do
  echo "== $v"
  env $v SGIGA_ASM_PROFILE=1 timeout 120 python - <<'PY' 2>&1 | grep asm-profile | tail -1
import sys; sys.path.insert(0, '.')
from paper_1707_09598_b200 import configs
from paper_1707_09598_b200.pipeline import Batch
from paper_1707_09598_b200.scheduler import make_spec
cfg = configs.get_config('cfg5')
b = Batch(make_spec(tuple(cfg.plan.terms), cfg.problem, cfg.quad_points))
for _ in range(2): b.assemble()
b.close()
PY
  env $v timeout 300 python bench.py --config cfg5 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['rooflines']
print('assembly ms', round(r['assembly']['ms'],3), 'step', round(d['ms_per_step'],3))"
done
