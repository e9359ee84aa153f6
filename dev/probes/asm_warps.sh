#!/bin/bash
# block-0 per-warp work cycles of the 3-D assembly (cfg5 / cfg5_tensor / cfg2)
for c in ${CFGS:-cfg5}; do
SGIGA_ASM_PROFILE=1 CFG=$c timeout 120 python - <<'PY' 2>&1 | grep asm-profile | tail -2
import os, sys; sys.path.insert(0, '.')
from paper_1707_09598_b200 import configs
from paper_1707_09598_b200.pipeline import Batch
from paper_1707_09598_b200.scheduler import make_spec
cfg = configs.get_config(os.environ['CFG'])
b = Batch(make_spec(tuple(cfg.plan.terms), cfg.problem, cfg.quad_points))
for _ in range(2): b.assemble()
b.close()
PY
done
