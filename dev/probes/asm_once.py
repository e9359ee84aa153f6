"""GPU probe (not a test): one assembly of a configuration (for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1707_09598_b200 import configs  # noqa: E402
from paper_1707_09598_b200.pipeline import Batch  # noqa: E402
from paper_1707_09598_b200.scheduler import make_spec  # noqa: E402

cfg = configs.get_config(sys.argv[1] if len(sys.argv) > 1 else "cfg5")
b = Batch(make_spec(tuple(cfg.plan.terms), cfg.problem, cfg.quad_points))
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 1):
    b.assemble()
b.close()
