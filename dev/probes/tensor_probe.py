"""GPU probe: cfg5's full tensor 2^6 comparison solve through one Batch --
phase times, kernel-group times, iterations and residuals."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_1707_09598_b200 import configs  # noqa: E402
from paper_1707_09598_b200.pipeline import Batch  # noqa: E402
from paper_1707_09598_b200.scheduler import make_spec  # noqa: E402

cfg = configs.get_config(sys.argv[1] if len(sys.argv) > 1 else "cfg5_tensor")
b = Batch(make_spec(tuple(cfg.plan.terms), cfg.problem, cfg.quad_points))
pts = cfg.points(4096)
for k in range(3):
    t0 = time.perf_counter()
    try:
        v = b.run(pts)
    except Exception as e:  # noqa: BLE001
        print("run failed:", type(e).__name__, e)
        break
    dt = time.perf_counter() - t0
    ms, ln = b.phase_stats()
    kt = np.zeros(7, dtype=np.float32)
    import ctypes as ct
    b.lib.sgiga_kernel_times(b.h, kt.ctypes.data_as(ct.POINTER(ct.c_float)))
    print(f"pass {k}: wall {dt*1e3:.1f} ms phases {ms} launches {ln} kernels(tab,met,asm,pcg,pcg2,post,comb) {kt}")
    print("iters", b.iters[:8], "relres", b.relres[:8])
b.close()
