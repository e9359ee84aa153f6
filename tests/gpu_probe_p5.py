"""GPU probe (not a test): assemble a small degree-4 3-D plan through the
fast kernel; run under compute-sanitizer to localise faults."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1707_09598_b200 import configs
from paper_1707_09598_b200.pipeline import Batch
from paper_1707_09598_b200.scheduler import make_spec

cfg = configs.get_config("cfg5")
terms = (((1, 1, 4), 1), ((2, 3, 2), 1), ((3, 1, 1), 1), ((1, 2, 1), 1))
if len(sys.argv) > 1 and sys.argv[1] == "full":
    terms = tuple(cfg.plan.terms)[:12]
spec = make_spec(terms, cfg.problem, cfg.quad_points)
b = Batch(spec)
b.assemble()
print("assembled ok", os.environ.get("SGIGA_NO_TMA"))
b.close()
