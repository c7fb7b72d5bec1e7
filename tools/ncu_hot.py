"""Hottest SASS instructions (by stall samples) of one kernel in an ncu report, with their
neighbourhood: python tools/ncu_hot.py <rep> <kernel-regex> [top]"""
import csv
import io
import subprocess
import sys

rep, krx = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{krx}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = next(i for i, r in enumerate(rows) if "Source" in r and "Instructions Executed" in r)
hdr = rows[h]
si, ii = hdr.index("Source"), hdr.index("Instructions Executed")
ss = hdr.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[h + 1:]:
    if len(r) <= ii:
        continue
    try:
        data.append((int(r[ss] or 0), int(r[ii] or 0), r[0], r[si].strip()))
    except ValueError:
        break
tot = sum(d[0] for d in data) or 1
print(f"{len(data)} instructions, {tot} stall samples")
for s, n, addr, src in sorted(data, reverse=True)[:top]:
    print(f"{100 * s / tot:5.1f}%  exec {n:>10}  {addr[-6:]}  {src[:90]}")
