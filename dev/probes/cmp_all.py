"""GPU probe: tiled vs pencil stencils of EVERY component (max entry error)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1707_09598_b200 import configs  # noqa: E402
from paper_1707_09598_b200.pipeline import Batch  # noqa: E402
from paper_1707_09598_b200.scheduler import make_spec  # noqa: E402
name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
cfg = configs.get_config(name)
spec = make_spec(tuple(cfg.plan.terms), cfg.problem, cfg.quad_points)
bs = {}
for mode in ("tile", "pencil"):
    os.environ["SGIGA_ASM_PENCIL"] = "1" if mode == "pencil" else "0"
    bs[mode] = Batch(spec)
    bs[mode].assemble()
worst = []
for c in range(len(spec.terms)):
    A1, b1 = bs["tile"].export_csr(c)
    A2, b2 = bs["pencil"].export_csr(c)
    assert np.array_equal(A1.indptr, A2.indptr) and np.array_equal(A1.indices, A2.indices)
    sc = np.abs(A2.data).max()
    ea = np.abs(A1.data - A2.data).max() / sc
    eb = np.abs(b1 - b2).max() / max(np.abs(b2).max(), 1e-300)
    # row sums (constants in the kernel of the stiffness away from the boundary)
    rs1 = np.abs(A1 @ np.ones(A1.shape[1])).max() / sc
    rs2 = np.abs(A2 @ np.ones(A2.shape[1])).max() / sc
    worst.append((ea, eb, rs1, rs2, c, spec.terms[c][0]))
worst.sort(reverse=True)
for w in worst[:12]:
    print("dA %.2e db %.2e rowsum tile %.2e pencil %.2e comp %d %s" % w)
print("median dA %.2e" % np.median([w[0] for w in worst]))
