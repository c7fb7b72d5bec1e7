"""Per-source-line instruction counts and stall samples from an ncu report (needs -lineinfo).

    python tools/ncu_lines.py <rep> <kernel-regex> [top]
"""
import csv
import io
import subprocess
import sys

rep, krx = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda",
                      "--kernel-name", f"regex:{krx}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = next(i for i, r in enumerate(rows) if "Source" in r and "Instructions Executed" in r)
hdr = rows[h]
si, ii = hdr.index("Source"), hdr.index("Instructions Executed")
ss = hdr.index("Warp Stall Sampling (All Samples)")
li = hdr.index("#") if "#" in hdr else 0
data = []
for r in rows[h + 1:]:
    if len(r) <= ii:
        continue
    try:
        n, s = int(r[ii] or 0), int(r[ss] or 0)
    except ValueError:
        continue
    data.append((n, s, r[li], r[si].strip()[:110]))
tot = sum(d[0] for d in data) or 1
tots = sum(d[1] for d in data) or 1
print(f"total warp-instructions {tot}  stall samples {tots}")
for d in sorted(data, reverse=True)[:top]:
    print(f"{d[0]:>11} {100 * d[0] / tot:5.1f}%  stall {100 * d[1] / tots:5.1f}%  L{d[2]:>5} | {d[3]}")
