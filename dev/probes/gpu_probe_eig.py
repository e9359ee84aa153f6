"""GPU probe (not a test): per-phase cycles of k_fd_eigen (SGIGA_FD_PROFILE=1)."""
import os
import sys

os.environ["SGIGA_FD_PROFILE"] = "1"
sys.path.insert(0, ".")
from paper_1707_09598_b200 import configs  # noqa: E402
from paper_1707_09598_b200.pipeline import Batch  # noqa: E402
from paper_1707_09598_b200.scheduler import make_spec  # noqa: E402

for name in sys.argv[1:] or ["cfg2"]:
    cfg = configs.get_config(name)
    spec = make_spec(tuple(cfg.plan.terms), cfg.problem, cfg.quad_points)
    b = Batch(spec)
    b.assemble()
    it, rr = b.solve(rtol=1e-13)
    print(name, "iters", it.tolist(), "relres max", rr.max())
    b.close()
