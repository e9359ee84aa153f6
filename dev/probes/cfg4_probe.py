"""GPU probe: cfg4 (multipatch L-shape, uniform and graded) -- session set-up
and per-solve wall times, iteration counts."""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1707_09598_b200 import configs  # noqa: E402
from paper_1707_09598_b200.multipatch import MultipatchSession  # noqa: E402

for name in ("cfg4", "cfg4_graded"):
    cfg = configs.get_multipatch_config(name)
    t0 = time.perf_counter()
    s = MultipatchSession(cfg.plan, cfg.problem)
    t1 = time.perf_counter()
    print(f"{name}: session set-up {1e3*(t1-t0):.1f} ms", flush=True)
    for k in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s.solve()
        t1 = time.perf_counter()
        print(f"{name} solve {k}: {1e3*(t1-t0):.2f} ms  interior iters max {int(s.iters.max())} "
              f"sum {int(s.iters.sum())}  boundary iters max {int(s.bnd_iters.max())}", flush=True)
    sol = s.solution()
    print(name, "L2/H1", sol.error_norms((8, 8), 3))
    sol.close()
