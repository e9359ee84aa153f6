#!/bin/bash
# 3-D assembly: parity subset, then cfg5 / cfg2 / tensor assembly times + block-0 stage profile
python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_r2.py -m gpu -q -p no:cacheprovider -x \
  -k "cfg5 or cfg2 or tensor or permutation or assembl or tma" 2>&1 | tail -2
for c in ${CFGS:-cfg5 cfg2 cfg5_tensor}; do
  timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['rooflines']
print('$c', 'step', round(d['ms_per_step'],3), 'assembly', round(r['assembly']['ms'],3), round(r['assembly'].get('frac',0),3))"
done
SGIGA_ASM_PROFILE=1 timeout 120 python - <<'PY' 2>&1 | grep asm-profile | tail -1
import sys; sys.path.insert(0, '.')
from paper_1707_09598_b200 import configs
from paper_1707_09598_b200.pipeline import Batch
from paper_1707_09598_b200.scheduler import make_spec
cfg = configs.get_config('cfg5')
b = Batch(make_spec(tuple(cfg.plan.terms), cfg.problem, cfg.quad_points))
for _ in range(2): b.assemble()
b.close()
PY
