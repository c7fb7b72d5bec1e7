"""Determinism probe of the O(1) path on the virtual-band test input (development tool):
the same call repeated must be bit-identical; prints the window-vs-whole max difference."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1605_02178_b200 as gc
from synth import config_image
for W in (333, 334):
    img = config_image("c5", H=400, W=W)
    t = torch.from_numpy(img).cuda()
    for sigma_s in (6.0, 16.0):
        ref = gc.filter(t, sigma_s, 55.0, 12, op=2)
        nd = 0
        for _ in range(20):
            o = gc.filter(t, sigma_s, 55.0, 12, op=2)
            nd += int(not torch.equal(o, ref))
        R = math.ceil(3 * sigma_s)
        bands = [0, 130, 260, 400]
        dmax, wnd = 0.0, 0
        for k in range(3):
            r0, r1 = bands[k], bands[k + 1]
            segs = ([(t[r0 - R:r0].clone(), r0 - R)] if k > 0 else []) + [(t[r0:r1].clone(), r0)] + \
                   ([(t[r1:r1 + R].clone(), r1)] if k < 2 else [])
            parts = [gc.filter_window(segs, 400, r0, r1 - r0, sigma_s, 55.0, 12, op=2) for _ in range(10)]
            wnd += sum(int(not torch.equal(p, parts[0])) for p in parts)
            dmax = max(dmax, float((parts[0] - ref[r0:r1]).abs().max()))
        print(f"W={W} sigma_s={sigma_s}: whole-image repeats differing {nd}/20, window repeats differing {wnd}/30, "
              f"window vs whole max-abs {dmax:.3e}", flush=True)
