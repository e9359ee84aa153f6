"""GPU probe: per-group kernel times of full passes (Batch.run) of a configuration."""
import ctypes as ct
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1707_09598_b200 import configs  # noqa: E402
from paper_1707_09598_b200.pipeline import Batch  # noqa: E402
from paper_1707_09598_b200.scheduler import make_spec  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
cfg = configs.get_config(name)
b = Batch(make_spec(tuple(cfg.plan.terms), cfg.problem, cfg.quad_points))
pts = cfg.points()
best = None
for _ in range(4):
    v = b.run(pts)
    kt = np.zeros(7, dtype=np.float32)
    b.lib.sgiga_kernel_times(b.h, kt.ctypes.data_as(ct.POINTER(ct.c_float)))
    best = kt.copy() if best is None else np.minimum(best, kt)
b.close()
print(f"{name}: metric {best[1]:.3f} assembly {best[2]:.3f} pcg {best[3] + best[4]:.3f} combine {best[6]:.3f} ms"
      f"  checksum {float(np.sum(v)):.17g}")
