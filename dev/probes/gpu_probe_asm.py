"""GPU probe (not a test): assembly phase profile for one config."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["SGIGA_ASM_PROFILE"] = "1"
from paper_1707_09598_b200 import configs
from paper_1707_09598_b200.pipeline import Batch
from paper_1707_09598_b200.scheduler import make_spec
cfg = configs.get_config(sys.argv[1])
b = Batch(make_spec(tuple(cfg.plan.terms), cfg.problem, cfg.quad_points))
print("pencils", len(b.spec.terms))
for _ in range(2):
    b.assemble()
b.close()
