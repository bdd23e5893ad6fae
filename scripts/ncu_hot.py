"""Top stall locations of an ncu report (SASS source page), for profiles/ summaries.
usage: python scripts/ncu_hot.py report.ncu-rep [N]"""
import csv
import io
import os
import subprocess
import sys

NCU = "/usr/local/cuda/bin/ncu" if os.path.exists("/usr/local/cuda/bin/ncu") else "ncu"

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
out = subprocess.run([NCU, "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hdr]
ci = h.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[hdr + 1:]:
    if len(r) > ci:
        try:
            data.append((float(r[ci] or 0), r[0], r[1]))
        except ValueError:
            pass
tot = sum(d[0] for d in data) or 1
data.sort(reverse=True)
for s, addr, src in data[:top]:
    print(f"{100 * s / tot:5.1f}%  {addr}  {src[:100]}")
