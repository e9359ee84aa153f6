"""Per-CUDA-line warp-stall breakdown (top stall reasons per hot line) from an
ncu report (--import-source, -lineinfo).  Runs here.

    python profiles/stall_lines.py <report.ncu-rep> [top]
"""
import csv
import signal
import subprocess
import sys

signal.signal(signal.SIGPIPE, signal.SIG_DFL)
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
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
    n = f("Warp Stall Sampling (All Samples)")
    reasons = sorted(((f(k), k[6:]) for k in hdr[2:] if k.startswith("stall_") and "Not Issued" not in k),
                     reverse=True)
    lines.append((n, f"{fname}:{r[0]}", r[1], reasons))
tot = sum(x[0] for x in lines) or 1.0
for n, loc, src, reasons in sorted(lines, key=lambda x: -x[0])[:top]:
    br = " ".join(f"{k}={100 * v / n:.0f}%" for v, k in reasons[:4] if v > 0 and n > 0)
    print(f"{100 * n / tot:5.1f}% {loc:>24}  {src.strip()[:60]:60s} {br}")
