"""GPU probe (not a test): assemble a plan (default: a small degree-4 3-D
subset) through the fast kernel once; with SGIGA_ASM_PROFILE=1 the kernel
prints block 0's per-interval phase cycles.

    python tests/gpu_probe_p5.py [cfg2|cfg5|full]
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1707_09598_b200 import configs
from paper_1707_09598_b200.pipeline import Batch
from paper_1707_09598_b200.scheduler import make_spec

arg = sys.argv[1] if len(sys.argv) > 1 else "small"
cfg = configs.get_config("cfg2" if arg == "cfg2" else "cfg5")
terms = (((1, 1, 4), 1), ((2, 3, 2), 1), ((3, 1, 1), 1), ((1, 2, 1), 1))
if arg == "full":
    terms = tuple(cfg.plan.terms)[:12]
elif arg in ("cfg2", "cfg5"):
    terms = tuple(cfg.plan.terms)
spec = make_spec(terms, cfg.problem, cfg.quad_points)
b = Batch(spec)
b.assemble()
print("assembled ok", arg, os.environ.get("SGIGA_NO_TMA"))
b.close()
