"""GPU probe: per-component PCG iterations and solver class of a config."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_1707_09598_b200 import configs
from paper_1707_09598_b200.pipeline import Batch
from paper_1707_09598_b200.scheduler import make_spec
cfg = configs.get_config(sys.argv[1])
b = Batch(make_spec(tuple(cfg.plan.terms), cfg.problem, cfg.quad_points))
b.assemble()
it, rr = b.solve(rtol=1e-13)
for (beta, c), i, r in zip(cfg.plan.terms, it, rr):
    print(beta, int(i), f"{r:.1e}")
b.close()
