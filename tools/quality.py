"""Full-image quality of the GCF against the direct filter of eq. (1), both on the GPU
(MSE in dB = 10 log10 mean-square error; PSNR = 10 log10(255^2 / MSE)), at the
BASELINE configs' stated sigma_r and at their parity twins (R1), with timings
of both filters (the Table II analogue) and the guard count (R8).

    python tools/quality.py [--configs c1 c2 c3 c4 c5] [--c4-images 8]
"""
import argparse
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import paper_1605_02178_b200 as gc
from synth import CONFIGS, config_image

a = argparse.ArgumentParser()
a.add_argument("--configs", nargs="*", default=["c1", "c2", "c3", "c4", "c5"])
a.add_argument("--c4-images", type=int, default=8)
args = a.parse_args()


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        out = fn()
    e1.record()
    torch.cuda.synchronize()
    return out, e0.elapsed_time(e1) / reps


def mse_db(x, y):
    m = float(torch.mean((x.double() - y.double()) ** 2))
    return (10 * math.log10(m) if m > 0 else -math.inf), (10 * math.log10(255.0 ** 2 / m) if m > 0 else math.inf)


print("| cfg | image | sigma_s | N | sigma_r | kind | GCF vs direct MSE (dB) | PSNR (dB) | guarded px | GCF ms | direct ms | speed-up |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|")
for name in args.configs:
    c = CONFIGS[name]
    if name == "c4":
        x = torch.from_numpy(np.stack([config_image(c, index=i) for i in range(args.c4_images)])).cuda()
        shape = f"{args.c4_images}x{c.H}x{c.W}"
    else:
        x = torch.from_numpy(config_image(c)).cuda()
        shape = f"{c.H}x{c.W}"
    for s in c.sigma_s:
        for kind, sr in (("stated", c.sigma_r), ("twin", c.sigma_r_twin)):
            fb = torch.zeros(1, dtype=torch.int64, device="cuda")
            g, tg = timed(lambda: gc.filter(x, s, sr, c.N))
            gc.filter(x, s, sr, c.N, fallback=fb)
            reps = 1 if (name == "c5" or s >= 20) else 3
            d, td = timed(lambda: gc.bilateral_direct(x, s, sr), reps=reps)
            mdb, psnr = mse_db(g, d)
            print(f"| {name} | {shape} | {s:g} | {c.N} | {sr:g} | {kind} | {mdb:.2f} | {psnr:.2f} | {int(fb.item())} | "
                  f"{tg:.3f} | {td:.1f} | {td / tg:.0f}x |", flush=True)
    del x
    torch.cuda.empty_cache()
