"""Does the O(1) window/whole result depend on what the scratch pool held before? (development
tool)  Runs the virtual-band comparison on a fresh process, then again after other calls have
filled the pool with unrelated data."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1605_02178_b200 as gc
from synth import config_image

def probe(tag):
    img = config_image("c5", H=400, W=333)
    t = torch.from_numpy(img).cuda()
    for sigma_s in (6.0, 16.0):
        ref = gc.filter(t, sigma_s, 55.0, 12, op=2)
        R = math.ceil(3 * sigma_s)
        bands = [0, 130, 260, 400]
        d = []
        for k in range(3):
            r0, r1 = bands[k], bands[k + 1]
            segs = ([(t[r0 - R:r0].clone(), r0 - R)] if k > 0 else []) + [(t[r0:r1].clone(), r0)] + \
                   ([(t[r1:r1 + R].clone(), r1)] if k < 2 else [])
            part = gc.filter_window(segs, 400, r0, r1 - r0, sigma_s, 55.0, 12, op=2)
            d.append(float((part - ref[r0:r1]).abs().max()))
        print(f"{tag}: sigma_s={sigma_s} window vs whole max-abs per band {['%.2e' % x for x in d]}", flush=True)
    return ref

a = probe("fresh")
# fill the scratch pool with unrelated data: big FIR / O(1) / Deriche calls on other images
for cfg, H, W, op in (("c2", 1024, 1024, 1), ("c3", 2048, 2048, 2), ("c3", 1000, 999, 3), ("c1", 400, 333, 1)):
    x = torch.from_numpy(config_image(cfg, H=H, W=W)).cuda() * 3.0 + 1000.0
    for s in (5.0, 16.0):
        try:
            gc.filter(x, s, 55.0, 12, op=op)
        except Exception as e:
            print("fill call", cfg, op, s, e)
torch.cuda.synchronize()
b = probe("after fill")
