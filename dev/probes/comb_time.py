"""GPU probe: combine kernel-group time (cfg) and bitwise check against the per-thread kernel."""
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
spec = make_spec(tuple(cfg.plan.terms), cfg.problem, cfg.quad_points)
pts = cfg.points()
res = {}
for mode in ("default", "tiled", "perthread"):
    os.environ["SGIGA_COMBINE_TILED"] = "1" if mode == "tiled" else "0"
    os.environ["SGIGA_COMBINE_PERTHREAD"] = "1" if mode == "perthread" else "0"
    b = Batch(spec)
    b.assemble()
    b.solve()
    ts = []
    for _ in range(3):
        v = b.combine_points(pts)
        kt = np.zeros(7, dtype=np.float32)
        b.lib.sgiga_kernel_times(b.h, kt.ctypes.data_as(ct.POINTER(ct.c_float)))
        ts.append(kt[6])
    res[mode] = v
    b.close()
    print(f"{name} {mode}: combine {min(ts):.4f} ms")
print("default == perthread bitwise:", np.array_equal(res["default"], res["perthread"]),
      "tiled == perthread:", np.array_equal(res["tiled"], res["perthread"]))
