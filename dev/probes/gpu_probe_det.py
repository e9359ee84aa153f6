"""GPU probe (not a test): run-to-run determinism of each stage."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1707_09598_b200 import configs
from paper_1707_09598_b200.pipeline import Batch
from paper_1707_09598_b200.scheduler import make_spec
cfg = configs.get_config(sys.argv[1] if len(sys.argv) > 1 else "cfg2")
spec = make_spec(tuple(cfg.plan.terms), cfg.problem, cfg.quad_points)
runs = []
for rep in range(3):
    b = Batch(spec); b.assemble()
    mats = [b.export_csr(c) for c in range(len(cfg.plan))]
    it, rr = b.solve()
    runs.append((mats, it.copy(), b.coefficients()))
    b.close()
for r in range(1, 3):
    dm = [c for c in range(len(cfg.plan)) if not (np.array_equal(runs[0][0][c][0].data, runs[r][0][c][0].data)
                                                   and np.array_equal(runs[0][0][c][1], runs[r][0][c][1]))]
    print("run", r, "matrix/rhs differ in comps", dm, "iters equal", np.array_equal(runs[0][1], runs[r][1]),
          "coef equal", np.array_equal(runs[0][2], runs[r][2]))
print("iters", [x[1].tolist() for x in runs])
