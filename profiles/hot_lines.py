"""Aggregate an ncu report's per-line metrics (cuda,sass source view; needs
-lineinfo): warp-stall samples, barrier stalls and shared-memory excess
wavefronts (bank conflicts) per CUDA source line.  Runs here.

    python profiles/hot_lines.py <report.ncu-rep> [top]
"""
import csv
import signal
import subprocess
import sys

signal.signal(signal.SIGPIPE, signal.SIG_DFL)

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
fname, hdr, lines = "?", None, []
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r or not r[0].isdigit():
        continue
    d = dict(zip(hdr[2:], r[2:]))

    def f(k):
        try:
            return float(d.get(k, 0) or 0)
        except ValueError:
            return 0.0
    lines.append((f"{fname}:{r[0]}", r[1], f("Warp Stall Sampling (All Samples)"), f("stall_barrier"),
                  f("L1 Wavefronts Shared Excessive"), f("Instructions Executed")))
tot = sum(x[2] for x in lines) or 1.0
print(f"{'line':>26} {'stall%':>7} {'barrier':>8} {'smem-excess':>12} {'inst':>12}  source")
for loc, src, st, bar, ex, inst in sorted(lines, key=lambda x: -x[2])[:top]:
    print(f"{loc:>26} {100 * st / tot:7.2f} {bar:8.0f} {ex:12.0f} {inst:12.0f}  {src.strip()[:80]}")
print("top bank-conflict lines:")
for loc, src, st, bar, ex, inst in sorted(lines, key=lambda x: -x[4])[:8]:
    print(f"{loc:>26} {ex:12.0f}  {src.strip()[:90]}")
