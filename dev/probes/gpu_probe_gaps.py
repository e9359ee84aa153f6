"""GPU probe (not a test): where the step time goes between the kernels.

Compares, per step, the bench's outer CUDA events with the handle's phase
events (assemble / solve / combine) and the kernel-group events."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1707_09598_b200 import configs  # noqa: E402
from paper_1707_09598_b200.pipeline import Batch  # noqa: E402
from paper_1707_09598_b200.scheduler import make_spec  # noqa: E402
import ctypes as ct  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
cfg = configs.get_config(name)
spec = make_spec(tuple(cfg.plan.terms), cfg.problem, cfg.quad_points)
b = Batch(spec)
stream = torch.cuda.ExternalStream(b.stream_ptr)
pts = torch.from_numpy(cfg.points()).cuda()
out = torch.empty(pts.shape[0], dtype=torch.float64, device="cuda")
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
for _ in range(5):
    b.run_device(pts.data_ptr(), pts.shape[0], out.data_ptr())
torch.cuda.synchronize()
for mode in ("flush", "noflush"):
    outer, phases, kts, walls = [], [], [], []
    for k in range(20):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            if mode == "flush":
                flush.zero_()
            s.record(stream)
        t0 = time.perf_counter()
        b.run_device(pts.data_ptr(), pts.shape[0], out.data_ptr())
        walls.append(time.perf_counter() - t0)
        with torch.cuda.stream(stream):
            e.record(stream)
        torch.cuda.synchronize()
        outer.append(s.elapsed_time(e))
        ms, _ = b.phase_stats()
        phases.append(ms.copy())
        kt = np.zeros(7, dtype=np.float32)
        b.lib.sgiga_kernel_times(b.h, kt.ctypes.data_as(ct.POINTER(ct.c_float)))
        kts.append(kt)
    print(f"[{mode}] outer ms {np.median(outer):.4f}  wall ms {1e3 * np.median(walls):.4f}  "
          f"phases(asm,solve,comb) {np.median(phases, axis=0)}  sum {np.median(np.sum(phases, axis=1)):.4f}  "
          f"kernel groups {np.round(np.median(kts, axis=0), 4)} sum {np.median(np.sum(kts, axis=1)):.4f}")
b.close()
