"""Dynamic SASS opcode mix (warp-instructions executed) of one kernel in an ncu report.

    python tools/ncu_mix.py <rep> <kernel-regex> [top]
"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep, krx = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{krx}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = next(i for i, r in enumerate(rows) if "Source" in r and "Instructions Executed" in r)
hdr = rows[h]
si, ii = hdr.index("Source"), hdr.index("Instructions Executed")
ss = hdr.index("Warp Stall Sampling (All Samples)")
mix, stall = Counter(), Counter()
for r in rows[h + 1:]:
    if len(r) <= ii:
        continue
    ins = r[si].strip()
    if ins.startswith("@"):
        ins = ins.split(None, 1)[1]
    op = ins.split()[0].split(".")[0] if ins else "?"
    try:
        n, st = int(r[ii] or 0), int(r[ss] or 0)
    except ValueError:
        continue
    mix[op] += n
    stall[op] += st
tot, tots = sum(mix.values()) or 1, sum(stall.values()) or 1
print(f"total {tot} warp-instructions")
for op, n in mix.most_common(top):
    print(f"{op:10s} {n:>12} {100 * n / tot:5.1f}%   stall-samples {100 * stall[op] / tots:5.1f}%")
