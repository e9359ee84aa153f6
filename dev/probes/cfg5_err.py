"""GPU probe: cfg5 L2/H1 errors and PCG iterations (assembly variant from env)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1707_09598_b200 import configs, analysis as A  # noqa: E402
from paper_1707_09598_b200.pipeline import Batch  # noqa: E402
from paper_1707_09598_b200.scheduler import make_spec  # noqa: E402
cfg = configs.get_config("cfg5")
b = Batch(make_spec(tuple(cfg.plan.terms), cfg.problem, cfg.quad_points))
b.assemble()
for rtol in (1e-13,):
    it, rr = b.solve(rtol=rtol)
    sid = A.solution_id_of(cfg.problem.solution)
    l2, h1 = b.error_norms(cfg.grid().points_per_dir, cfg.grid().weights_per_dir, sid)
    print(os.environ.get("SGIGA_ASM_PENCIL", "0"), rtol, "l2 %.4e h1 %.4e" % (l2, h1), "iters", int(it.sum()), "max relres %.2e" % rr.max())
b.close()
