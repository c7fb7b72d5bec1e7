"""Quick per-kernel timing of gc.filter on a config (development tool, not the bench).

    python tools/time_ops.py c5 [--op 2] [--sigma-s 16] [--reps 10] [--H 4096 --W 4096]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import paper_1605_02178_b200 as gc
from synth import CONFIGS, config_image

a = argparse.ArgumentParser()
a.add_argument("cfg")
a.add_argument("--op", type=int, default=0)
a.add_argument("--sigma-s", type=float, nargs="*", default=None)
a.add_argument("--reps", type=int, default=10)
a.add_argument("--H", type=int, default=None)
a.add_argument("--W", type=int, default=None)
a.add_argument("--B", type=int, default=None)
args = a.parse_args()
c = CONFIGS[args.cfg]
B = args.B or c.batch
H, W = args.H or c.H, args.W or c.W
def _img(i):
    # within one gpurun call, repeated invocations reuse the generated image (scratch cache)
    import hashlib
    tag = hashlib.sha1(open(os.path.join(ROOT, "synth", "images.py"), "rb").read()).hexdigest()[:10]
    f = f"/tmp/gc_timeops_{tag}_{args.cfg}_{i}_{H}x{W}.npy"
    if os.path.exists(f):
        return np.load(f)
    a = config_image(c, index=i, H=H, W=W)
    np.save(f, a)
    return a


if B > 1:
    x = torch.from_numpy(np.stack([_img(i) for i in range(B)])).cuda()
else:
    x = torch.from_numpy(_img(0)).cuda()
out = torch.empty_like(x)
for s in (args.sigma_s or c.sigma_s):
    for op in ([1, 2] if args.op == 0 else [args.op]):
        if op == 1 and np.ceil(3 * s) > 1024:
            continue
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.reps)]
        for e in evs:
            for q in e:
                q.record()
        for _ in range(2):
            gc.filter(x, s, c.sigma_r, c.N, op=op, out=out)
        torch.cuda.synchronize()
        for k in range(args.reps):
            gc.filter(x, s, c.sigma_r, c.N, op=op, out=out, events=evs[k])
        torch.cuda.synchronize()
        row = np.median([e[0].elapsed_time(e[1]) for e in evs])
        col = np.median([e[1].elapsed_time(e[2]) for e in evs])
        px = B * H * W
        print(f"{args.cfg} {B}x{H}x{W} sigma_s={s:5.1f} N={c.N} op={'FIR' if op == 1 else 'O1 '}: "
              f"row {row:8.3f} ms  col {col:8.3f} ms  total {row + col:8.3f} ms  {px / (row + col) / 1e6:8.2f} Gpx/s",
              flush=True)
