"""Development probe: one c2 image as K concurrent row-band windows on K streams vs one call."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import paper_1605_02178_b200 as gc
from synth import CONFIGS, config_image

c = CONFIGS["c2"]
x = torch.from_numpy(config_image(c)).cuda()
H = x.shape[0]
R = 15
args = (5.0, 70.0, 8)
out = torch.empty_like(x)
flush = torch.empty(256 * 1024 * 1024 // 4, device="cuda")


def whole():
    gc.filter(x, *args, out=out)


def split(k, streams):
    cur = torch.cuda.current_stream()
    ev = torch.cuda.Event()
    ev.record(cur)
    rows = [H * i // k for i in range(k + 1)]
    done = []
    for i in range(k):
        s = streams[i]
        s.wait_event(ev)
        with torch.cuda.stream(s):
            gc.filter_window([(x, 0)], H, rows[i], rows[i + 1] - rows[i], *args, out=out[rows[i]:rows[i + 1]])
            e = torch.cuda.Event()
            e.record(s)
            done.append(e)
    for e in done:
        cur.wait_event(e)


streams = [torch.cuda.Stream() for _ in range(8)]
ref = None
for name, fn in [("whole", whole)] + [(f"split{k}", (lambda k=k: split(k, streams))) for k in (2, 3, 4)]:
    for _ in range(5):
        flush.zero_()
        fn()
    torch.cuda.synchronize()
    if ref is None:
        ref = out.clone()
    else:
        assert torch.equal(out, ref), name
    ts = []
    for _ in range(100):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    print(f"{name}: median {np.median(ts):.1f} us", flush=True)
