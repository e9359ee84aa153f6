"""GPU probe (not a test): FD vs Jacobi iteration counts and agreement."""
import os
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1707_09598_b200 import configs  # noqa: E402
from paper_1707_09598_b200.pipeline import Batch  # noqa: E402
from paper_1707_09598_b200.scheduler import make_spec  # noqa: E402

for name in sys.argv[1:] or ["cfg1", "cfg2", "cfg3"]:
    cfg = configs.get_config(name)
    spec = make_spec(tuple(cfg.plan.terms), cfg.problem, cfg.quad_points)
    out = {}
    for mode in ("fd", "jacobi"):
        os.environ["SGIGA_NO_FD"] = "1" if mode == "jacobi" else "0"
        b = Batch(spec)
        b.assemble()
        try:
            it, rr = b.solve(rtol=1e-13)
        except Exception as e:  # noqa: BLE001
            print(name, mode, "solve error", e)
            it, rr = b.iters, b.relres
        out[mode] = (b.coefficients(), it, rr)
        b.close()
    cf, itf, rrf = out["fd"]
    cj, itj, rrj = out["jacobi"]
    rel = np.linalg.norm(cf - cj) / np.linalg.norm(cj)
    print(f"{name}: fd iters {itf.tolist()}\n   jacobi iters {itj.tolist()}\n   fd relres max {rrf.max():.3e} "
          f"jacobi relres max {rrj.max():.3e} rel diff {rel:.3e}")
