"""Summarise ncu captures (made by profiles/capture.sh on the GPU box) into the
tracked text files under profiles/<round>/ and the per-launch DRAM traffic
table profiles/traffic.json that bench.py reports as roofline.traffic.

    python profiles/summarize.py gpurun_out/r01b profiles/r01

Reads `launches_<cfg>.csv` (gpu__time_duration of every launch of a
`bench.py --steps 1 --warmup 3` run) and `asm_<cfg>.ncu-rep` (`--set full`
of the first assembly launch).  Runs here (ncu -i needs no GPU).
"""
from __future__ import annotations

import csv
import io
import json
import os
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_active.max", "launch__grid_size", "launch__block_size",
    "launch__registers_per_thread", "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "smsp__inst_executed.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def _launch_table(path: str, cfg: str) -> str:
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr, rows = rows[0], rows[1:]
    iN, iV = hdr.index("Kernel Name"), hdr.index("Metric Value")
    iS = hdr.index("Stream") if "Stream" in hdr else None
    names = [r[iN].split("(")[0] for r in rows]
    # the last step = everything after the last occurrence of the first kernel
    # of a step (k_basis_tables opens every sgiga_run)
    starts = [i for i, n in enumerate(names) if n.endswith("k_basis_tables")]
    lo = starts[-1] if starts else 0
    sel = [(names[i], float(rows[i][iV].replace(",", "")), rows[i][iS] if iS is not None else "")
           for i in range(lo, len(rows))]
    tot = sum(v for _, v, _ in sel)
    out = [f"# ncu launch list, {cfg} bench step (python bench.py --config <workload> --steps 1 --warmup 3), last step",
           "# ncu --metrics gpu__time_duration.sum --clock-control none (serialised, cold-ish caches)",
           "# kernel, ns, share of the step's summed kernel time, stream (side streams overlap the main one)"]
    out += [f"{n:48s} {v:10.0f} {100 * v / tot:6.1f}%  stream {st}" for n, v, st in sel]
    out.append(f"{'total':48s} {tot:10.0f}")
    return "\n".join(out) + "\n"


def _full_summary(rep: str):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, val = rows[0], rows[1], rows[2]
    lines = [f"{'Kernel Name':60s} {val[hdr.index('Kernel Name')]}"]
    got = {}
    for k in KEYS:
        if k in hdr:
            i = hdr.index(k)
            lines.append(f"{k:60s} {val[i]} {units[i]}")
            try:
                got[k] = float(val[i].replace(",", "")) * UNIT.get(units[i], 1)
            except ValueError:
                pass
    st = []
    for i, h in enumerate(hdr):
        if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued"):
            try:
                st.append((float(val[i].replace(",", "")), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(v for v, _ in st) or 1.0
    lines.append("# warp-state samples (share of all samples)")
    lines += [f"  stall {n:28s} {100 * v / tot:5.1f}%" for v, n in sorted(st, reverse=True)[:8]]
    return "\n".join(lines) + "\n", got


def _hot_lines(rep: str, top: int = 15) -> str:
    here = os.path.dirname(os.path.abspath(__file__))
    out = subprocess.run([sys.executable, os.path.join(here, "hot_lines.py"), rep, str(top)],
                         capture_output=True, text=True).stdout
    return "# per-source-line warp-stall samples and shared-memory excess wavefronts (profiles/hot_lines.py)\n" + out


def main(src: str, dst: str) -> None:
    """Every launches_<workload>.csv -> launches_<workload>.txt; every
    <kernel>_<workload>.ncu-rep -> ncu_full_<kernel>_<workload>.txt (section
    metrics, warp-state samples, hot source lines); the assembly captures
    feed profiles/traffic.json (bench.py's roofline.traffic)."""
    os.makedirs(dst, exist_ok=True)
    tpath = os.path.join(os.path.dirname(os.path.abspath(__file__)), "traffic.json")
    traffic = {}   # rebuilt from the captures in src (one entry per workload and kernel group)
    for f in sorted(os.listdir(src)):
        path = os.path.join(src, f)
        if f.startswith("launches_") and f.endswith(".csv"):
            wl = f[len("launches_"):-4]
            open(os.path.join(dst, f"launches_{wl}.txt"), "w").write(_launch_table(path, wl))
        elif f.endswith(".ncu-rep"):
            stem = f[:-8]
            txt, got = _full_summary(path)
            head = f"# ncu --set full --clock-control none --import-source on, first launch ({stem})\n"
            open(os.path.join(dst, f"ncu_full_{stem}.txt"), "w").write(head + txt + _hot_lines(path))
            # per workload and kernel group (bench.py's rooflines keys): DRAM bytes of one launch
            groups = {"k_assemble_tile": "assembly", "k_stencil_box": "assembly", "k_assemble2d": "assembly",
                      "k_pcg_fdl": "pcg", "k_pcg_fdg": "pcg", "k_combine_points_tiled": "combine"}
            for kern, grp in groups.items():
                if stem.startswith(kern + "_") and "dram__bytes_read.sum" in got:
                    wl = stem[len(kern) + 1:]
                    traffic.setdefault(wl, {})[grp] = {
                        "kernel": kern,
                        "dram_bytes_per_launch": got["dram__bytes_read.sum"] + got.get("dram__bytes_write.sum", 0.0),
                        "source": os.path.join(os.path.basename(os.path.normpath(dst)), f"ncu_full_{stem}.txt"),
                    }
    json.dump(traffic, open(tpath, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
