import sys
sys.path.insert(0, ".")
from paper_1707_09598_b200 import configs  # noqa: E402
from paper_1707_09598_b200.multipatch import MultipatchSession  # noqa: E402
cfg = configs.get_multipatch_config(sys.argv[1] if len(sys.argv) > 1 else "cfg4")
s = MultipatchSession(cfg.plan, cfg.problem)
s.solve()
s.solve()
s.close()
