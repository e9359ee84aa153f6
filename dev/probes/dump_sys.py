"""GPU probe: dump a few components' assembled systems (exact bytes) to compare libraries."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1707_09598_b200 import configs  # noqa: E402
from paper_1707_09598_b200.pipeline import Batch  # noqa: E402
from paper_1707_09598_b200.scheduler import make_spec  # noqa: E402
name, out = sys.argv[1], sys.argv[2]
cfg = configs.get_config(name)
spec = make_spec(tuple(cfg.plan.terms), cfg.problem, cfg.quad_points)
b = Batch(spec)
b.assemble()
n = len(spec.terms)
d = {}
for c in sorted({0, n // 3, n // 2, n - 1}):
    A, r = b.export_csr(c)
    d[f"A{c}"] = A.data
    d[f"b{c}"] = r
np.savez(out, **d)
