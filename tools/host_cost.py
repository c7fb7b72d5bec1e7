"""Host-side cost of one gc_filter call (development probe): enqueue rate on a tiny image."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import ctypes
import torch

import paper_1605_02178_b200 as gc

x = torch.rand(64, 64, device="cuda") * 255
out = torch.empty_like(x)
for _ in range(20):
    gc.filter(x, 5.0, 70.0, 8, out=out)
torch.cuda.synchronize()
n = 2000
t0 = time.perf_counter()
for _ in range(n):
    gc.filter(x, 5.0, 70.0, 8, out=out)
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"python gc.filter: {(t1 - t0) / n * 1e6:.1f} us/call host")
# the C call alone, parameters prepared once
p, keep = gc._params(8, 5.0, 70.0)
L = gc._lib()
ip, op_, st = gc._dev_f32(x, "x"), gc._dev_f32(out, "o"), gc._stream(None)
t0 = time.perf_counter()
for _ in range(n):
    L.gc_filter(ip, 1, 64, 64, ctypes.byref(p), op_, st)
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"C gc_filter: {(t1 - t0) / n * 1e6:.1f} us/call host (back to back, may be GPU-bound)")
# one call at a time on an idle GPU
ts = []
for _ in range(200):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    L.gc_filter(ip, 1, 64, 64, ctypes.byref(p), op_, st)
    ts.append(time.perf_counter() - t0)
ts.sort()
print(f"C gc_filter on an idle GPU: median {ts[len(ts) // 2] * 1e6:.1f} us/call host")
big = torch.rand(1024, 1024, device="cuda") * 255
bo = torch.empty_like(big)
ib, ob = gc._dev_f32(big, "b"), gc._dev_f32(bo, "o")
ts = []
for _ in range(200):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    L.gc_filter(ib, 1, 1024, 1024, ctypes.byref(p), ob, st)
    ts.append(time.perf_counter() - t0)
ts.sort()
print(f"C gc_filter 1024^2 on an idle GPU: median {ts[len(ts) // 2] * 1e6:.1f} us/call host")
