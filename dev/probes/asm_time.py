"""GPU probe: assembly kernel-group time of a configuration (env picks the kernel)."""
import ctypes as ct
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1707_09598_b200 import configs  # noqa: E402
from paper_1707_09598_b200.pipeline import Batch  # noqa: E402
from paper_1707_09598_b200.scheduler import make_spec  # noqa: E402

name = sys.argv[1]
R = int(sys.argv[2]) if len(sys.argv) > 2 else 1   # replicated batch (R copies of the plan)
cfg = configs.get_config(name)
b = Batch(make_spec(tuple(cfg.plan.terms) * R, cfg.problem, cfg.quad_points))
ts = []
for _ in range(3):
    b.assemble()
    kt = np.zeros(7, dtype=np.float32)
    b.lib.sgiga_kernel_times(b.h, kt.ctypes.data_as(ct.POINTER(ct.c_float)))
    ts.append(kt[2])
b.close()
print(f"{name} x{R} pencil={os.environ.get('SGIGA_ASM_PENCIL', '0')}: assembly {min(ts):.3f} ms (metric {kt[1]:.3f})")
