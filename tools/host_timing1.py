"""Host wall time of gc_filter_host (the e2e call) for one config and the current
GC_HOST_CHUNKS setting: python tools/host_timing1.py <cfg> [B]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import paper_1605_02178_b200 as gc
from synth import CONFIGS, config_image

name = sys.argv[1]
c = CONFIGS[name]
B = int(sys.argv[2]) if len(sys.argv) > 2 else 1
img = np.stack([config_image(c, index=i) for i in range(B)]) if B > 1 else config_image(c)
hin = torch.from_numpy(img).pin_memory()
hout = torch.empty_like(hin).pin_memory()
for _ in range(3):
    gc.filter_host(hin.numpy(), c.sigma_s[0], c.sigma_r, c.N, out=hout.numpy())
n = 10 if img.size > 1e8 else 50
t0 = time.perf_counter()
for _ in range(n):
    gc.filter_host(hin.numpy(), c.sigma_s[0], c.sigma_r, c.N, out=hout.numpy())
dt = (time.perf_counter() - t0) / n
print(f"{name} B={B} chunks={os.environ.get('GC_HOST_CHUNKS', 'auto')}: {dt * 1e6:.0f} us/call  "
      f"{img.size / dt / 1e9:.2f} Gpx/s", flush=True)
