"""c1 (256x256, sigma_s = 3, N = 5) is launch-latency bound: time gc.filter captured in a CUDA
graph and replayed: microseconds per call, plain stream launches beside it."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import paper_1605_02178_b200 as gc
from synth import CONFIGS, config_image

c = CONFIGS["c1"]
x = torch.from_numpy(config_image(c)).cuda()
out = torch.empty_like(x)
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for _ in range(3):
        gc.filter(x, c.sigma_s[0], c.sigma_r, c.N, out=out)
torch.cuda.synchronize()
n = 1000
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(n):
    gc.filter(x, c.sigma_s[0], c.sigma_r, c.N, out=out)
e1.record()
torch.cuda.synchronize()
plain = e0.elapsed_time(e1) / n * 1e3
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    for _ in range(10):
        gc.filter(x, c.sigma_s[0], c.sigma_r, c.N, out=out)
torch.cuda.synchronize()
g.replay()
torch.cuda.synchronize()
e0.record()
for _ in range(n // 10):
    g.replay()
e1.record()
torch.cuda.synchronize()
graph = e0.elapsed_time(e1) / n * 1e3
ref = gc.filter(x, c.sigma_s[0], c.sigma_r, c.N)
torch.cuda.synchronize()
assert torch.equal(ref, out)
px = c.H * c.W
print(f"c1 256x256 sigma_s=3 N=5: stream launches {plain:.2f} us/call ({px / plain / 1e3:.2f} Gpx/s); "
      f"CUDA graph replay (10 calls/graph) {graph:.2f} us/call ({px / graph / 1e3:.2f} Gpx/s)")
