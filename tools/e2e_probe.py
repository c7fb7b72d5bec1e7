"""Why the bench's e2e number differs from a bare gc_filter_host loop (development probe):
times the same call with and without the L2 flush before it, by host wall clock and by events."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import paper_1605_02178_b200 as gc
from synth import CONFIGS, config_image

c = CONFIGS["c2"]
img = config_image(c)
hin = torch.from_numpy(img).pin_memory()
hout = torch.empty_like(hin).pin_memory()
hin_np, hout_np = hin.numpy(), hout.numpy()
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
args = (c.sigma_s[0], c.sigma_r, c.N)
for _ in range(5):
    gc.filter_host(hin_np, *args, out=hout_np)
n = 50
for mode in ["bare", "flush", "flush+sync", "events", "events+flush"] * 2:
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tw = te = 0.0
    for _ in range(n):
        if "flush" in mode:
            flush.zero_()
        if "sync" in mode:
            torch.cuda.synchronize()
        if "events" in mode:
            e0.record()
        t0 = time.perf_counter()
        gc.filter_host(hin_np, *args, out=hout_np)
        tw += time.perf_counter() - t0
        if "events" in mode:
            e1.record()
            e1.synchronize()
            te += e0.elapsed_time(e1) / 1e3
    print(f"{mode:14s} wall {tw / n * 1e6:7.1f} us" + (f"  events {te / n * 1e6:7.1f} us" if te else ""), flush=True)
