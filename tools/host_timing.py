"""Host-side timing of gc_filter_host (the e2e call) for a config, by chunk count."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import paper_1605_02178_b200 as gc
from synth import CONFIGS, config_image

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
c = CONFIGS[name]
B = int(sys.argv[2]) if len(sys.argv) > 2 else 1
img = np.stack([config_image(c, index=i) for i in range(B)]) if B > 1 else config_image(c)
hin = torch.from_numpy(img).pin_memory()
hout = torch.empty_like(hin).pin_memory()
x = hin.cuda()
for K in ["1", "2", "4", "8", "auto"]:
    if K == "auto":
        os.environ.pop("GC_HOST_CHUNKS", None)
    else:
        os.environ["GC_HOST_CHUNKS"] = K
    for _ in range(3):
        gc.filter_host(hin.numpy(), c.sigma_s[0], c.sigma_r, c.N, out=hout.numpy())
    n = 20
    t0 = time.perf_counter()
    for _ in range(n):
        gc.filter_host(hin.numpy(), c.sigma_s[0], c.sigma_r, c.N, out=hout.numpy())
    dt = (time.perf_counter() - t0) / n
    print(f"{name} B={B} chunks={K}: {dt * 1e6:.0f} us/call  {img.size / dt / 1e9:.2f} Gpx/s", flush=True)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20):
    gc.filter(x, c.sigma_s[0], c.sigma_r, c.N)
torch.cuda.synchronize()
print(f"device-only gc.filter: {(time.perf_counter() - t0) / 20 * 1e6:.0f} us/call (host wall)")
t0 = time.perf_counter()
for _ in range(20):
    hout.copy_(x, non_blocking=True)
    x.copy_(hin, non_blocking=True)
torch.cuda.synchronize()
print(f"torch H2D+D2H copies: {(time.perf_counter() - t0) / 20 * 1e6:.0f} us/iter")
