"""GPU probe (not a test): small-path PCG convergence per cluster size."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1707_09598_b200 import configs
from paper_1707_09598_b200.pipeline import Batch
from paper_1707_09598_b200.scheduler import make_spec
for name in ("cfg2", "cfg3"):
    cfg = configs.get_config(name)
    spec = make_spec(tuple(cfg.plan.terms), cfg.problem, cfg.quad_points)
    for k in sys.argv[1:]:
        os.environ["SGIGA_CLUSTER_K"] = k
        b = Batch(spec); b.assemble()
        try:
            it, rr = b.solve(maxit=3000)
            print(name, "K", k, "ok its", it.tolist())
        except Exception as e:  # noqa
            print(name, "K", k, "FAIL", str(e)[:80], b.iters.tolist() if b.iters is not None else None)
        b.close()
