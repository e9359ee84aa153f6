"""Probe (not a test): phase and kernel-group times of repeated cfg runs."""
import ctypes as ct
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1707_09598_b200 import configs  # noqa: E402
from paper_1707_09598_b200.pipeline import Batch  # noqa: E402
from paper_1707_09598_b200.scheduler import make_spec  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
cfg = configs.get_config(name)
spec = make_spec(tuple(cfg.plan.terms), cfg.problem, cfg.quad_points)
b = Batch(spec)
pts = np.random.default_rng(0).random((32768, spec.d))
for it in range(6):
    b.run(pts)
    ms, ln = b.phase_stats()
    kt = np.zeros(7, dtype=np.float32)
    b.lib.sgiga_kernel_times(b.h, kt.ctypes.data_as(ct.POINTER(ct.c_float)))
    print(f"run {it}: phases asm/solve/comb ms {np.round(ms, 4)}  groups tab/met/asm/pcg/pcg2/post/comb {np.round(kt, 4)}")
b.close()
