"""Top SASS instructions by warp-stall samples from an ncu report's source
page (ncu -i REP --page source --csv), with the dominant stall reason."""
import csv
import subprocess
import sys

rep, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
iS, iN = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
data = []
for k, r in enumerate(rows[2:]):
    if len(r) < len(hdr):
        continue
    try:
        n = float(r[iN] or 0)
    except ValueError:
        continue
    st = max(stall_cols, key=lambda i: float(r[i] or 0))
    data.append((n, k, r[0], r[iS], hdr[st]))
tot = sum(d[0] for d in data) or 1
for n, k, a, s, st in sorted(data, reverse=True)[:top]:
    print(f"{100 * n / tot:5.1f}%  #{k:5d} {a:>6s}  {s[:60]:60s} {st}")
