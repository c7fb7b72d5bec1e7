"""Does running the passes of different row bands concurrently (2 streams) beat one whole-image
call?  Development probe: times gc_filter on the c5 image vs K row bands through gc_filter_window
alternating over two streams (the halo rows are read from the same device image).

    python tools/band_overlap.py [K ...]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import paper_1605_02178_b200 as gc
from synth import CONFIGS, config_image

c = CONFIGS["c5"]
H, W = c.H, c.W
f = f"/tmp/gc_band_overlap_c5.npy"
img = np.load(f) if os.path.exists(f) else config_image(c)
if not os.path.exists(f):
    np.save(f, img)
x = torch.from_numpy(img).cuda()
out = torch.empty_like(x)
s_main = torch.cuda.current_stream()
streams = [torch.cuda.Stream(), torch.cuda.Stream()]


def whole():
    gc.filter(x, 16.0, c.sigma_r, c.N, out=out)


def bands(K):
    cuts = [H * k // K for k in range(K + 1)]
    ev0 = torch.cuda.Event()
    ev0.record(s_main)
    for k in range(K):
        st = streams[k % 2]
        st.wait_event(ev0)
        r0, r1 = cuts[k], cuts[k + 1]
        gc.filter_window([(x, 0)], H, r0, r1 - r0, 16.0, c.sigma_r, c.N, out=out[r0:r1], stream=st)
    for st in streams:
        e = torch.cuda.Event()
        e.record(st)
        s_main.wait_event(e)


def timeit(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


t = timeit(whole)
print(f"whole image: {t:.3f} ms  {H * W / t / 1e6:.2f} Gpx/s", flush=True)
ref = out.clone()
for K in [int(a) for a in sys.argv[1:]] or [2, 4, 8]:
    tb = timeit(lambda: bands(K))
    d = (out - ref).abs().max().item()
    print(f"{K} bands / 2 streams: {tb:.3f} ms  {H * W / tb / 1e6:.2f} Gpx/s  (max diff vs whole {d:.2e})", flush=True)
