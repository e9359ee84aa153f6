#!/usr/bin/env python
"""Throughput benchmark of the batched assemble -> PCG -> combine pipeline.

Metric (BASELINE.json): components solved/s & DoF/s (assemble+CG+combine),
% of FP64/HBM roofline.  One "step" = the whole hot path on one plan:
assemble every component, solve every component (PCG to 1e-13: FD-
preconditioned for the small components, Jacobi for the large ones),
combine at the configuration's evaluation points.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2]
    python bench.py --impl reference ...     # reference CPU path (oracle port)

Workload: BASELINE configs[4] (cfg5: 3-D unit cube, p=4 C^3, w=12, 136
components, 1.43 M dofs, 32768 random points, seed 4) -- the largest
configuration that fits one GPU, as the tier rules ask when the metric
names no config -- unless --config says otherwise.  Inputs are synthetic
and fully defined by the config (no dataset).

`value` = components/s with every input resident in HBM (device timing,
CUDA events on the library's stream, L2 flushed before each step).
`e2e`   = the same metric through the public API with host buffers
(PlanSession.run: H2D of the problem inputs + points, pipeline, D2H of
the combined values), wall clock.
N > 1 (torchrun): --mode split (default) shards ONE plan's components over
the ranks (LPT on a modelled cost), with one NCCL all-gather of per-
component point values and the plan-order sum on the device (strong
scaling); --mode replicas runs one independent plan per rank (weak).
"""
from __future__ import annotations

import argparse
import ctypes as ct
import json
import os
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "components solved/s & DoF/s (assemble+CG+combine), % of FP64/HBM roofline"
UNIT = "components/s"


def canonical_work(plan, p, q, d, levels_to_dims):
    """Per-component canonical counts: rows, reference nnz,
    elements, assembly FLOPs F_el (sum-factorised stiffness + load)."""
    P = p + 1
    F_el = 2 * d * d * sum(P ** (d + k + 1) for k in range(1, d + 1)) + 2 * d * P ** (d + 1)
    out = []
    for beta, _ in plan.terms:
        n = levels_to_dims(beta)
        m = [x - 2 for x in n]
        nnz = 1
        for mm in m:
            nnz *= sum(min(mm - 1, i + p) - max(0, i - p) + 1 for i in range(mm))
        nel = int(np.prod([2**b for b in beta]))
        W = 2 * p + 1
        stored = int(np.prod(m)) * int(np.prod([min(max(mm, 1), W) for mm in m]))   # stencil slots kept on device
        out.append(dict(rows=int(np.prod(m)), nnz=int(nnz), dofs=int(np.prod(n)), nel=nel, flops=nel * F_el,
                        stored=stored))
    return out


class NvmlClockSampler:
    """SM clocks + throttle reasons sampled through NVML on a background thread
    every ~1 ms; only samples taken between begin() and end() (the timed
    region, host clock) are reported, so short regions still get samples."""

    def __init__(self, index=0):
        import threading

        import pynvml as N
        self.N = N
        N.nvmlInit()
        vis = [v for v in os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",") if v.strip()]
        phys = int(vis[index]) if index < len(vis) and vis[index].strip().isdigit() else index
        self.h = N.nvmlDeviceGetHandleByIndex(phys)
        self.max_sm = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
        self.rows, self.t0, self.t1 = [], None, None
        self.run = True
        self.th = threading.Thread(target=self._loop, daemon=True)
        self.th.start()

    def _loop(self):
        N = self.N
        while self.run:
            t = time.perf_counter()
            try:
                sm = N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM)
                rs = N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                break
            self.rows.append((t, sm, rs))
            time.sleep(0.0005)

    def begin(self):
        self.t0 = time.perf_counter()

    def end(self):
        self.t1 = time.perf_counter()

    def stop(self):
        self.run = False
        self.th.join()
        N = self.N
        sel = [r for r in self.rows if self.t0 is not None and self.t0 <= r[0] <= (self.t1 or r[0])]
        bits = {"hw_slowdown": N.nvmlClocksEventReasonHwSlowdown,
                "hw_thermal_slowdown": N.nvmlClocksEventReasonHwThermalSlowdown,
                "sw_thermal_slowdown": N.nvmlClocksEventReasonSwThermalSlowdown,
                "sw_power_cap": N.nvmlClocksEventReasonSwPowerCap}
        reasons = sorted({k for _, _, rs in sel for k, bit in bits.items() if rs & bit})
        sm = [r[1] for r in sel]
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": float(self.max_sm),
                "reasons": reasons, "samples": len(sel), "source": "nvml"}


def clock_sampler(index=0):
    try:
        return NvmlClockSampler(index)
    except Exception:
        return ClockSampler(index)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons while the timed region runs
    (fallback when NVML is unavailable)."""

    def begin(self):
        pass

    def end(self):
        pass

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        self.proc.terminate()
        self.proc.wait()
        self.f.flush()
        rows = [r.split(",") for r in Path(self.f.name).read_text().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm = [float(r[0]) for r in rows if r[0].strip().replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if len(r) > 4 + i and "Active" in r[4 + i]
                          and "Not" not in r[4 + i]})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def fp64_peak_tflops():
    lib = ct.CDLL(str(ROOT / "paper_1707_09598_b200" / "libsgiga_peaks.so"))
    lib.sgiga_fp64_peak.argtypes = [ct.c_double, ct.POINTER(ct.c_double), ct.POINTER(ct.c_double)]
    tf, ms = ct.c_double(), ct.c_double()
    if lib.sgiga_fp64_peak(0.5, ct.byref(tf), ct.byref(ms)) != 0:
        return None
    return float(tf.value)


def _ncu_traffic() -> dict:
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "traffic.json")
    try:
        with open(path) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return json.loads(p.read_text()), "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def config_dict(cfg, ws, replicas=1, mode="replicas", rtol=1e-13):
    """The workload description -- identical in both arms (same keys, same
    values), so the driver can check that they ran the same work."""
    from paper_1707_09598_b200.scheduler import make_spec

    spec = make_spec(tuple(cfg.plan.terms), cfg.problem, cfg.quad_points)
    dofs = int(sum(int(np.prod([2**b + spec.degree for b in beta])) for beta, _ in cfg.plan.terms))
    if ws == 1:
        par = "single GPU"
    elif mode == "split":
        par = f"components of one plan LPT-sharded over {ws} GPUs + one all-gather at the combine"
    else:
        par = f"{ws} independent plan replicas (one per GPU)"
    return {"workload": cfg.name, "d": spec.d, "degree": spec.degree, "level_w": cfg.plan.level,
            "components": len(cfg.plan) * replicas, "points": cfg.n_points, "dofs": dofs * replicas,
            "quad_points": spec.quad_points, "rtol": rtol, "replicas": replicas, "parallelism": par}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ---------------------------------------------------------------------------
# reference arm: the reference's CPU algorithm (oracle port) on host cores
# ---------------------------------------------------------------------------
def reference_step(cfg, threads, terms=None):
    """One full reference pass on the host cores: every component of the plan
    assembled (element kernel in the reference's loop order) and solved
    directly, then the per-point combine -- scheduler.run_plan
    (scheduler.py:74-96) + the per-point idiom (test_acceptance.py:224-230)."""
    from oracle import oracle as O
    from paper_1707_09598_b200.scheduler import make_spec

    terms = tuple(cfg.plan.terms) if terms is None else terms
    spec = make_spec(terms, cfg.problem, cfg.quad_points)
    orc = O.Oracle(spec, threads=threads)
    pts = cfg.points()
    t0 = time.perf_counter()
    orc.run_plan(O.SOLVER_DIRECT, threads=threads)
    orc.combine_points(pts, threads=threads)
    dt = time.perf_counter() - t0
    dofs = int(orc.dof_offsets[-1])
    return len(terms), dofs, dt


def run_reference(args, cfg):
    """--impl reference: the reference's CPU algorithm (oracle port, every
    host thread) on the SAME workload as the GPU arm -- the full plan every
    step.  A cfg5 step is ~100 s on 16 cores, so K + W full steps do not fit
    the driver's arm limit: the arm times full steps until --ref-budget
    seconds are spent (at least one) and says so in the line; nothing is
    sampled."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    threads = len(os.sched_getaffinity(0))
    os.environ.setdefault("OMP_NUM_THREADS", str(threads))
    # warm-up: one small component (thread pool, page-in); a full warm-up
    # step would cost as much as a timed one and the CPU path has no JIT
    small = (min(cfg.plan.terms, key=lambda t: sum(t[0])),)
    reference_step(cfg, threads, small)
    times, ncomp, dofs = [], 0, 0
    t_start = time.perf_counter()
    for k in range(args.steps):
        ncomp, dofs, dt = reference_step(cfg, threads)
        times.append(dt)
        spent = time.perf_counter() - t_start
        if spent + dt > args.ref_budget:
            break
    t = float(np.mean(times))
    value = ncomp / t
    conf = config_dict(cfg, ws, mode=args.mode, rtol=args.rtol)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "steps_timed": len(times), "ms_per_step": 1e3 * t,
        "higher_is_better": True, "scaling": "strong" if (ws > 1 and args.mode == "split") else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (BASELINE config recipe; seeded points)",
        "config": conf,
        "dof_per_s": dofs / t,
        "timing": (f"{len(times)} full-plan step(s) timed (wall clock, host); a step = all {ncomp} components "
                   f"+ the {cfg.n_points}-point combine; further steps skipped once --ref-budget "
                   f"{args.ref_budget:.0f} s was spent; warm-up = one small component"),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "cpu_model": cpu_model(),
                         "sample": f"full plan: {ncomp} of {len(cfg.plan)} components (assemble + direct solve, "
                                   f"OpenMP over components) + {cfg.n_points}-point per-point combine, per step"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_multipatch(args, name):
    """BASELINE configs[3] (cfg4 / cfg4_graded): the L-shape from 3 patches,
    p = 2, w = 9, 15 components glued C0 with Dirichlet lifting
    (multipatch.MultipatchSession).  A step = assemble every patch, glue,
    project the Dirichlet data, solve (batched cluster CSR PCG), expand, then
    evaluate the 4 096 points on every patch."""
    import torch

    from paper_1707_09598_b200.configs import get_multipatch_config
    from paper_1707_09598_b200.multipatch import MultipatchSession

    ws, rank, local = dist_env()
    if rank != 0:
        return 0
    torch.cuda.set_device(local)
    cfg = get_multipatch_config(name)
    pts = cfg.points()
    n_comp = len(cfg.plan)
    if args.impl == "reference":   # the multipatch oracle (numpy restatement), one step
        from oracle import multipatch_oracle as MO
        from paper_1707_09598_b200.multipatch import _PatchProblem
        from paper_1707_09598_b200.scheduler import make_spec
        prob = cfg.problem
        specs = [make_spec(tuple(cfg.plan.terms), _PatchProblem(pt, prob.forcing, prob.degree, prob.regularity),
                           cfg.quad_points, knot_rule=prob.knot_rules[pi]) for pi, pt in enumerate(prob.patches)]
        t0 = time.perf_counter()
        MO.run_plan(specs, prob, cfg.quad_points)
        dt = time.perf_counter() - t0
        line = {"impl": "reference", "metric": METRIC, "value": n_comp / dt, "unit": UNIT, "n_gpus": ws,
                "steps": 1, "warmup": 0, "ms_per_step": 1e3 * dt, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic (BASELINE config recipe)",
                "config": {"workload": name, "d": 2, "degree": 2, "level_w": 9, "components": n_comp, "patches": 3,
                           "points": cfg.n_points, "rtol": args.rtol},
                "cpu_baseline": {"value": n_comp / dt, "unit": UNIT, "cores": 1, "kind": "port",
                                 "cpu_model": cpu_model(),
                                 "sample": "oracle/multipatch_oracle.py (dense numpy restatement), full plan, one step"},
                "e2e": {"value": n_comp / dt, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return 0
    sess = MultipatchSession(cfg.plan, cfg.problem, cfg.quad_points, rtol=args.rtol)
    for _ in range(max(args.warmup, 3)):
        sess.solve()
    torch.cuda.synchronize()
    sampler = clock_sampler(local)
    time.sleep(0.01)
    sampler.begin()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    t0 = time.perf_counter()
    for s, e in ev:
        s.record()
        sess.solve()
        vals = [sess.batches[pi].combine_points(pts) for pi in range(3)]
        e.record()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / args.steps
    sampler.end()
    clocks = sampler.stop()
    ms = float(np.mean([s.elapsed_time(e) for s, e in ev]))
    line = {"metric": METRIC, "value": n_comp / (ms * 1e-3), "unit": UNIT, "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (BASELINE config recipe)",
            "config": {"workload": name, "d": 2, "degree": 2, "level_w": 9, "components": n_comp, "patches": 3,
                       "points": cfg.n_points, "rtol": args.rtol},
            "timing": "CUDA events around each step (the session's host synchronisations included)",
            "e2e": {"value": n_comp / wall, "unit": UNIT, "h2d_bytes_per_step": int(3 * pts.nbytes),
                    "d2h_bytes_per_step": int(3 * pts.shape[0] * 8), "ms_per_step": 1e3 * wall,
                    "path": "MultipatchSession.solve + Batch.combine_points (host points in, host values out)"},
            "pcg_iterations": {"interior_max": int(sess.iters.max()), "interior_sum": int(sess.iters.sum()),
                               "boundary_max": int(sess.bnd_iters.max())},
            "clocks": clocks, "cpu_baseline": None}
    sol = sess.solution()
    line["errors_l2_h1"] = list(sol.error_norms((8, 8), cfg.quad_points))
    print(json.dumps(line), flush=True)
    sol.close()
    return 0


def run_split(args, cfg):
    """N > 1, --mode split: ONE plan's components LPT-sharded over the ranks
    (distributed.DistributedPlan): per step every rank assembles + solves its
    share and evaluates it at the points into a device buffer, one NCCL
    all-gather, the plan-order sum on the device.  Strong scaling: the value
    is the whole plan's components / the max-over-ranks step time."""
    import torch
    import torch.distributed as dist

    from paper_1707_09598_b200.distributed import DistributedPlan, component_cost_model

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if "MASTER_ADDR" not in os.environ:   # --split-world1 outside torchrun
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29533", RANK="0", WORLD_SIZE="1")
    dist.init_process_group("nccl", device_id=dev)
    dp = DistributedPlan(cfg.plan, cfg.problem, cfg.quad_points, rtol=args.rtol)
    pts_h = cfg.points()
    npts = pts_h.shape[0]
    pts_d = torch.from_numpy(pts_h).to(dev)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)   # 256 MB > L2
    for _ in range(max(args.warmup, 3)):
        dp.step(pts_d)
    torch.cuda.synchronize()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    dist.barrier()
    torch.cuda.synchronize()
    sampler = clock_sampler(local)
    time.sleep(0.01)
    sampler.begin()
    for k in range(args.steps):
        flush.zero_()
        starts[k].record()
        vals = dp.step(pts_d)
        ends[k].record()
    torch.cuda.synchronize()
    sampler.end()
    clocks = sampler.stop()
    total_ms = float(sum(s.elapsed_time(e) for s, e in zip(starts, ends)))
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_per_step = float(t.item()) / args.steps
    # e2e: host points in (pinned, H2D inside the step), host values out
    pin = torch.empty(pts_h.shape, dtype=torch.float64, pin_memory=True)
    pin.copy_(torch.from_numpy(pts_h))
    out_h = torch.empty(npts, dtype=torch.float64, pin_memory=True)
    dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        pts_step = pin.to(dev, non_blocking=True)
        out_h.copy_(dp.step(pts_step), non_blocking=True)
        torch.cuda.current_stream().synchronize()
    e2e_s = (time.perf_counter() - t0) / args.steps
    t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_s = float(t.item())
    same = bool(torch.equal(vals.cpu(), out_h))
    n_comp = len(cfg.plan)
    cost = component_cost_model(cfg.plan.terms, cfg.problem.degree, cfg.plan.d)
    loads = [float(cost[p].sum()) for p in dp.parts]
    launches = 0
    if dp.batch is not None:
        _, ln = dp.batch.phase_stats()
        launches = int(ln.sum()) + 2    # + the all-gather's NCCL kernel and the plan-order sum
    lt = torch.tensor([launches], dtype=torch.float64, device=dev)
    dist.all_reduce(lt)
    if rank == 0:
        line = {
            "metric": METRIC, "value": n_comp / (ms_per_step * 1e-3), "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (BASELINE config recipe; seeded points)",
            "config": config_dict(cfg, ws, 1, "split", args.rtol),
            "timing": "CUDA events around each step on every rank, max over ranks; 256 MB L2 flush before "
                      "every timed step (outside the events)",
            "e2e": {"value": n_comp / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(pts_h.nbytes),
                    "d2h_bytes_per_step": int(npts * 8), "ms_per_step": 1e3 * e2e_s,
                    "matches_device_run_bitwise": same,
                    "path": "pinned points H2D -> DistributedPlan.step (assemble + solve + per-component "
                            "combine, NCCL all-gather, plan-order sum) -> pinned values D2H, per step"},
            "partition": {"components_per_rank": [len(p) for p in dp.parts],
                          "modelled_load_s": loads, "model": "distributed.component_cost_model (LPT)"},
            "gpu_launches": int(lt.item()) * args.steps,
            "clocks": clocks,
            "cpu_baseline": None,
        }
        print(json.dumps(line), flush=True)
    dp.close()
    dist.destroy_process_group()
    return 0


def run_sgiga(args, cfg):
    import torch
    import torch.distributed as dist

    from paper_1707_09598_b200.pipeline import Batch
    from paper_1707_09598_b200.scheduler import PlanSession, make_spec

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    R = max(1, args.replicas)
    terms = tuple(cfg.plan.terms) * R       # replicated batch: R copies, one launch
    spec = make_spec(terms, cfg.problem, cfg.quad_points)
    batch = Batch(spec)
    stream = torch.cuda.ExternalStream(batch.stream_ptr)
    pts_h = cfg.points()
    npts = pts_h.shape[0]
    pts_d = torch.from_numpy(pts_h).to(f"cuda:{local}")
    out_d = torch.empty(npts, dtype=torch.float64, device=f"cuda:{local}")
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=f"cuda:{local}")   # 256 MB > L2

    def step():   # assemble + solve + combine, one library call, one sync
        batch.run_device(pts_d.data_ptr(), npts, out_d.data_ptr(), rtol=args.rtol)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    kt_acc = np.zeros(7)
    launches = 0
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler = clock_sampler(local)
    time.sleep(0.01)
    sampler.begin()
    # timed passes are enqueued back to back (sgiga_run_async: no host round
    # trip between them); every pass does the full assemble + solve +
    # combine, and sgiga_run_wait reports the last one's convergence verdict
    for k in range(args.steps):
        with torch.cuda.stream(stream):
            flush.zero_()          # L2 flush, outside the timed events
            starts[k].record(stream)
        batch.run_device_async(pts_d.data_ptr(), npts, out_d.data_ptr(), rtol=args.rtol)
        with torch.cuda.stream(stream):
            ends[k].record(stream)
    batch.run_wait()
    torch.cuda.synchronize()
    sampler.end()
    clocks = sampler.stop()
    kt = np.zeros(7, dtype=np.float32)     # kernel groups of the last pass (same work every pass)
    batch.lib.sgiga_kernel_times(batch.h, kt.ctypes.data_as(ct.POINTER(ct.c_float)))
    kt_acc += kt * args.steps
    _, ln = batch.phase_stats()
    launches += int(ln.sum()) * args.steps
    step_ms = np.array([s.elapsed_time(e) for s, e in zip(starts, ends)])
    total_ms = float(step_ms.sum())
    if ws > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
        dist.barrier()
    ms_per_step = total_ms / args.steps
    n_comp = len(terms)
    iters = batch.iters.copy()
    vals = out_d.cpu().numpy()

    # ---- canonical work and rooflines ---------------------------------------
    dims = [tuple(int(x) for x in row) for row in batch.dims]
    lookup = {tuple(b): dims[i] for i, (b, _) in enumerate(terms)}

    class _Terms:   # canonical_work only reads .terms
        pass
    plan_r = _Terms()
    plan_r.terms = terms
    work = canonical_work(plan_r, spec.degree, spec.quad_points, spec.d, lambda b: lookup[tuple(b)])
    dofs = sum(w["dofs"] for w in work)
    kt = kt_acc / args.steps   # ms per launch group per step
    cg_bytes = sum(int(it) * (8 * w["nnz"] + 104 * w["rows"]) for it, w in zip(iters, work))
    # the sweeps the FD-PCG actually makes: one stencil read per iteration
    # plus the true-residual SpMV (linsolve.py:49-53), over the stored slots
    # (Kronecker box systems above the small-component kernel's 2048 rows:
    # the true residual rides in the iteration sweeps, no sweep of its own)
    def _sweeps(it, w):
        return int(it) + (0 if (_box and w["rows"] > 2048 and it >= 1) else 1)
    _akind = ct.c_int32(0)
    batch.lib.sgiga_assembly_kind(batch.h, ct.byref(_akind))
    _box = int(_akind.value) == 2
    cg_sweep_bytes = sum(_sweeps(it, w) * 8 * w["stored"] + int(it) * 104 * w["rows"] for it, w in zip(iters, work))
    asm_flops = sum(w["flops"] for w in work)
    ex = ct.c_double(0.0)   # FP64 operations the assembly launch executed (host count of its work items)
    batch.lib.sgiga_assembly_flops(batch.h, ct.byref(ex))
    asm_exec = float(ex.value)
    akind = ct.c_int32(0)   # 0 row/2-D/generic kernels, 1 tiled 3-D, 2 Kronecker box assembly
    batch.lib.sgiga_assembly_kind(batch.h, ct.byref(akind))
    asm_kind = {0: "row", 1: "tiled", 2: "box"}[int(akind.value)]
    # box assembly: 1-D bands -> ONE store pass over the live stencil entries
    # (HBM-store bound), the load by three sum-factorisation stages of f det w
    nqp = sum(w["nel"] for w in work) * spec.quad_points ** spec.d
    asm_box_bytes = sum(8 * w["stored"] + 16 * w["rows"] for w in work) + 8 * nqp
    d = spec.d
    comb_flops_pt = 0
    P = spec.degree + 1
    levels_per_axis = [len({b[k] for b, _ in cfg.plan.terms}) for k in range(d)]
    comb_flops_pt = sum(L * (2 * spec.degree + 5 * spec.degree * (spec.degree + 1) // 2) for L in levels_per_axis) \
        + n_comp * (2 * sum(P**j for j in range(1, d + 1)) + 2)
    comb_flops = comb_flops_pt * npts
    comb_bytes = npts * (8 * d + 8) + 8 * dofs
    peaks, peak_kind = measured_peaks()
    hbm_peak = float(peaks["hbm_gbs"])
    fp64 = fp64_peak_tflops() if rank == 0 else None
    cg_ms = kt[3] + kt[4]
    groups = {
        "pcg": dict(ms=cg_ms, bound="hbm", achieved=cg_bytes / (cg_ms * 1e-3) / 1e9 if cg_ms > 0 else 0.0,
                    peak=hbm_peak, unit="GB/s", traffic_algorithmic_bytes=cg_bytes,
                    stencil_sweep_bytes=cg_sweep_bytes,
                    stencil_sweep_gbs=cg_sweep_bytes / (cg_ms * 1e-3) / 1e9 if cg_ms > 0 else 0.0,
                    note="achieved/frac: SURVEY B_it = iterations x (8 nnz + 104 n); stencil_sweep_*: the stored "
                         "stencil read once per iteration + once for the true residual (box systems on the line-FD / "
                         "whole-GPU kernels: the true residual is fused into the iteration sweeps)",
                    peak_source=f"{peak_kind} MEASURED_PEAKS.json hbm_gbs"),
        "assembly": (dict(ms=kt[2], bound="hbm", kernel="k_stencil_box + k_rhs_box_stage x3 (Kronecker box assembly)",
                          achieved=asm_box_bytes / (kt[2] * 1e-3) / 1e9 if kt[2] > 0 else 0.0,
                          peak=hbm_peak, unit="GB/s", algorithmic_bytes=asm_box_bytes,
                          canonical_flops=asm_flops,
                          canonical_tflops=asm_flops / (kt[2] * 1e-3) / 1e12 if kt[2] > 0 else 0.0,
                          note="axis-aligned box geometry: the stiffness is a Kronecker sum of 1-D mass/stiffness "
                               "bands, so the kernel does not execute SURVEY 8(d)'s per-element FLOPs (canonical_tflops "
                               "is what the canonical count would imply); its floor is the store of the stencil: "
                               "bytes = 8 x live stencil slots + 16 x rows (load, diagonal) + 8 x quadrature points "
                               "(f det w read by the load stages)",
                          peak_source=f"{peak_kind} MEASURED_PEAKS.json hbm_gbs")
                     if asm_kind == "box" else
                     dict(ms=kt[2], bound="fp64", kernel=f"stencil assembly ({asm_kind})",
                          achieved=asm_flops / (kt[2] * 1e-3) / 1e12 if kt[2] > 0 else 0.0,
                          peak=fp64, unit="TFLOP/s", canonical_flops=asm_flops,
                          executed_flops=asm_exec,
                          executed_tflops=asm_exec / (kt[2] * 1e-3) / 1e12 if kt[2] > 0 and asm_exec > 0 else None,
                          peak_source="DFMA micro-benchmark on this GPU (tools/fp64_peak.cu)")),
        "combine": dict(ms=kt[6], bound="fp64", achieved=comb_flops / (kt[6] * 1e-3) / 1e12 if kt[6] > 0 else 0.0,
                        peak=fp64, unit="TFLOP/s", canonical_flops=comb_flops,
                        hbm_gbs=comb_bytes / (kt[6] * 1e-3) / 1e9 if kt[6] > 0 else 0.0,
                        peak_source="DFMA micro-benchmark on this GPU (tools/fp64_peak.cu)"),
        "metric": dict(ms=kt[1], note="geometry/metric/load per quadrature point"),
        "tables": dict(ms=kt[0]),
        "post": dict(ms=kt[5], note="residual check + expand"),
    }
    for g in groups.values():
        if g.get("peak"):
            g["frac"] = g["achieved"] / g["peak"]
            if g.get("executed_tflops"):
                g["executed_frac"] = g["executed_tflops"] / g["peak"]
    dom = max(("pcg", "assembly", "combine"), key=lambda k: groups[k]["ms"])
    G = groups[dom]
    tr = _ncu_traffic().get(args.config, {}).get(dom, {}) if R == 1 else {}
    if G["bound"] == "hbm":
        # dominant group bound by HBM: the FD-PCG (stencil sweeps) or the box assembly (stencil store)
        if dom == "pcg":
            kname = ("FD-preconditioned CG: k_pcg_fdl (one cluster per component) / k_pcg_fdg (whole GPU) / "
                     "k_pcg_fd (small components, side stream)")
            abytes = cg_bytes
        else:
            kname, abytes = G.get("kernel", dom), G.get("algorithmic_bytes")
        roofline = {"bound": "hbm", "achieved": G["achieved"], "peak": G["peak"], "unit": "GB/s",
                    "frac": G["frac"], "traffic": tr.get("dram_bytes_per_launch"),
                    "traffic_source": tr.get("source"), "traffic_kernel": tr.get("kernel"),
                    "group": dom, "kernel": kname,
                    "algorithmic_bytes_per_launch": abytes, "peak_source": G["peak_source"]}
    else:
        # DRAM bytes of one launch of the dominant kernel from the committed
        # `ncu --set full` capture (profiles/capture.sh -> profiles/summarize.py)
        roofline = {"bound": "tensor", "achieved": G["achieved"], "peak": G["peak"], "unit": "TFLOP/s",
                    "frac": G.get("frac"),
                    "traffic": tr.get("dram_bytes_per_launch"),
                    "traffic_source": tr.get("source"),
                    "kernel": dom,
                    "note": "FP64 CUDA-core bound; 'tensor' slot holds the measured DFMA peak. achieved = the "
                            "canonical sum-factorised FLOPs of SURVEY 8(d) (F_el per element) / kernel time; the "
                            "tiled kernel shares stage-1 contractions and plane windows across the rows of a tile, "
                            "so it executes fewer FLOPs than the canonical count (frac can exceed 1); "
                            "executed_* = the FLOPs the launch actually executed",
                    "executed_flops_per_launch": G.get("executed_flops"),
                    "executed_tflops": G.get("executed_tflops"),
                    "executed_frac": G.get("executed_frac"),
                    "peak_source": G["peak_source"]}

    # ---- end to end through the public API, host buffers ---------------------
    if R == 1:
        sess = PlanSession(cfg.plan, cfg.problem, cfg.quad_points, rtol=args.rtol)
    else:   # replicated batch: the same public call on the replicated spec
        class _Sess:
            def __init__(self):
                self.b = Batch(spec)
                self.h2d_input_bytes = int(sum(a.nbytes for a in self.b._keep.values()))

            def run(self, pts):
                return self.b.run(pts, args.rtol)

            def close(self):
                self.b.close()
        sess = _Sess()
    pin = torch.empty(pts_h.shape, dtype=torch.float64, pin_memory=True)
    pin.copy_(torch.from_numpy(pts_h))
    pts_pinned = pin.numpy()
    for _ in range(max(args.warmup, 3)):
        sess.run(pts_pinned)
    # (a) latency: one synchronous call per step (H2D points, pass, D2H values)
    if ws > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        v_e2e = sess.run(pts_pinned)
    sync_s = (time.perf_counter() - t0) / args.steps
    # (b) throughput (the e2e value): the same pass submitted back to back on
    # page-locked host buffers -- every step still copies its points H2D and
    # its values D2H inside the pass; one wait at the end, then every step's
    # output is checked bitwise against the synchronous call
    async_ok = hasattr(sess, "submit")
    if async_ok:
        outs = [torch.empty(npts, dtype=torch.float64, pin_memory=True) for _ in range(args.steps)]
        for k in range(max(args.warmup, 3)):
            sess.submit(pts_pinned, outs[k % len(outs)].numpy())
        sess.wait()
        if ws > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for k in range(args.steps):
            sess.submit(pts_pinned, outs[k].numpy())
        sess.wait()
        e2e_s = (time.perf_counter() - t0) / args.steps
        async_ok = all(np.array_equal(o.numpy(), v_e2e) for o in outs)
    else:
        e2e_s = sync_s
    if ws > 1:
        t = torch.tensor([e2e_s, sync_s], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s, sync_s = float(t[0].item()), float(t[1].item())
    h2d = pts_h.nbytes              # the problem descriptor is uploaded once, at session open
    desc_bytes = sess.h2d_input_bytes
    d2h = npts * 8 + n_comp * (4 + 8) + 64
    consistent = bool(np.array_equal(v_e2e, vals))
    sess.close()

    # ---- CPU baseline (rank 0, N = 1) ---------------------------------------
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        threads = len(os.sched_getaffinity(0))
        nc, cdofs, dt = reference_step(cfg, threads)
        cpu = {"value": nc / dt, "unit": UNIT, "cores": threads, "kind": "port", "cpu_model": cpu_model(),
               "sample": f"full plan: {nc} of {len(cfg.plan)} components (assemble + direct solve) + {npts}-point "
                         f"combine, 1 step, oracle/sgiga_oracle.c (C restatement of the reference), OpenMP "
                         f"{threads} threads"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": ws * n_comp / (ms_per_step * 1e-3), "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (BASELINE config recipe; seeded points)",
            "config": config_dict(cfg, ws, R, args.mode, args.rtol),
            "timing": "CUDA events on the library stream, K passes enqueued back to back, 256 MB L2 flush "
                      "before every timed pass (outside the events); max over ranks",
            "dof_per_s": ws * dofs / (ms_per_step * 1e-3),
            "e2e": {"value": ws * n_comp / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "ms_per_step": 1e3 * e2e_s,
                    "mode": ("pipelined: PlanSession.submit per step (pinned points H2D + pass + values D2H), "
                             "one wait, every step's output checked bitwise; no L2 flush (warm, as a user sees it)")
                    if hasattr(sess, "submit") else "synchronous PlanSession.run per step",
                    "all_steps_match": bool(async_ok) if hasattr(sess, "submit") else None,
                    "sync_ms_per_step": 1e3 * sync_s, "sync_value": ws * n_comp / sync_s,
                    "matches_device_run_bitwise": consistent,
                    "descriptor_bytes_uploaded_at_open": int(desc_bytes),
                    "path": "PlanSession.submit -> sgiga_run_host_async (pinned host points in, pinned host values out); sync: PlanSession.run -> sgiga_run"},
            "roofline": roofline,
            "rooflines": {k: {kk: (float(vv) if isinstance(vv, (np.floating, float)) else vv) for kk, vv in g.items()}
                          for k, g in groups.items()},
            "pcg_iterations": {"sum": int(iters.sum()), "max": int(iters.max())},
            "gpu_launches": int(launches),
            "clocks": clocks,
            "fp64_peak_tflops_measured": fp64,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    batch.close()
    if ws > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="sgiga", choices=["sgiga", "reference"])
    ap.add_argument("--config", default="cfg5")
    ap.add_argument("--rtol", type=float, default=1e-13)
    ap.add_argument("--ref-budget", type=float, default=600.0,
                    help="reference arm: stop timing further full-plan steps after this many seconds")
    ap.add_argument("--mode", default="split", choices=["replicas", "split"],
                    help="N > 1: one plan split over the GPUs (strong, default) or independent plan replicas per "
                         "GPU (weak)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--split-world1", action="store_true", help=argparse.SUPPRESS)   # test the split path at N = 1
    ap.add_argument("--replicas", type=int, default=1,
                    help="replicated batch: R copies of the plan in one launch (SURVEY 8(d) roofline scaling)")
    args = ap.parse_args()
    from paper_1707_09598_b200.configs import get_config

    if args.config in ("cfg4", "cfg4_graded"):
        return run_multipatch(args, args.config)
    cfg = get_config(args.config)
    if args.impl == "reference":
        return run_reference(args, cfg)
    if args.mode == "split" and (dist_env()[0] > 1 or args.split_world1):
        return run_split(args, cfg)
    return run_sgiga(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
