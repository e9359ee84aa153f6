"""GPU probe (not a test): tiled vs per-pencil 3-D assembly -- kernel time of
the assembly group and the stencil difference on a few components.

    python dev/probes/tile_probe.py cfg5 [reps]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1707_09598_b200 import configs  # noqa: E402
from paper_1707_09598_b200.pipeline import Batch  # noqa: E402
from paper_1707_09598_b200.scheduler import make_spec  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = configs.get_config(name)
spec = make_spec(tuple(cfg.plan.terms), cfg.problem, cfg.quad_points)
pick = sorted(set([0, 1, len(spec.terms) // 3, len(spec.terms) // 2, len(spec.terms) - 1]))
mats = {}
for mode in ("pencil", "tile"):
    os.environ["SGIGA_ASM_PENCIL"] = "1" if mode == "pencil" else "0"
    os.environ["SGIGA_ASM_PROFILE"] = "0"
    b = Batch(spec)
    ts = []
    for _ in range(reps):
        b.assemble()
        kt = np.zeros(7, dtype=np.float32)
        import ctypes as ct
        b.lib.sgiga_kernel_times(b.h, kt.ctypes.data_as(ct.POINTER(ct.c_float)))
        ts.append(kt.copy())
    mats[mode] = [b.export_csr(c) for c in pick]
    b.close()
    ts = np.array(ts)
    print(f"{name} {mode}: kernel groups (ms, last rep) {np.round(ts[-1], 3).tolist()}  asm min {ts[:, 0].min():.3f}")
    sys.stdout.flush()
os.environ["SGIGA_ASM_PENCIL"] = "0"
os.environ["SGIGA_ASM_PROFILE"] = "1"
b = Batch(spec)
b.assemble()
b.close()
for c, (A1, b1), (A2, b2) in zip(pick, mats["pencil"], mats["tile"]):
    same = np.array_equal(A1.indptr, A2.indptr) and np.array_equal(A1.indices, A2.indices)
    da = np.linalg.norm(A1.data - A2.data) / max(np.linalg.norm(A1.data), 1e-300) if same else float("nan")
    db = np.linalg.norm(b1 - b2) / max(np.linalg.norm(b1), 1e-300)
    print(f"comp {c} {spec.terms[c][0]}: pattern {'same' if same else 'DIFFERENT'} dA {da:.2e} db {db:.2e}")
