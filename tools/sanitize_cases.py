"""Small invocations of every libgc device path, run against the bounds-checked library
(compute-sanitizer is not available on the B200 pool):

    GC_LIB_PATH=paper_1605_02178_b200/libgc_check.so python tools/sanitize_cases.py

Every global-memory access of the kernels is range-checked in that build (gc_device.cuh GC_CHK);
this prints the number of out-of-bounds accesses the cases made and exits non-zero if any (or if
a call failed or an output is non-finite).  Output buffers also carry NaN guard margins that must
be untouched.  tests/test_gpu_bounds.py runs it.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import paper_1605_02178_b200 as gc
from synth import config_image

OP_FIR, OP_O1, OP_DR = 1, 2, 3


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def main():
    torch.cuda.set_device(0)
    outs = []
    checked = "bounds-check" in gc.version()
    # whole images: the three operators, even and odd widths (TMA vs cp.async O(1) column paths)
    for (H, W) in [(64, 96), (61, 77), (1, 33), (40, 1)]:
        x = dev(config_image("c2", H=max(H, 2), W=max(W, 2))[:H, :W])
        for op in (OP_FIR, OP_O1, OP_DR):
            for s in (2.0, 9.0):
                outs.append(gc.filter(x, s, 70.0, 8, op=op))
        outs.append(gc.gaussian(x, 3.0, op=OP_O1))
        outs.append(gc.filter(x, 2.0, 70.0, 8, fp64=True))
        outs.append(gc.bilateral_direct(x, 2.0, 30.0))
    # large N: G > 1 lanes per column in the legacy O(1) column pass, FIR with NP > 8
    x = dev(config_image("c2", H=70, W=90))
    outs.append(gc.filter(x, 9.0, 200.0, 20, op=OP_O1))
    outs.append(gc.filter(x, 3.0, 200.0, 20, op=OP_FIR))
    # batches
    xb = dev(np.stack([config_image("c4", index=i, H=48, W=64) for i in range(3)]))
    for op in (OP_FIR, OP_O1, OP_DR):
        outs.append(gc.filter(xb, 4.0, 85.0, 6, op=op))
    # virtual row bands (gc_filter_window, three segments) incl. interior windows
    img = config_image("c5", H=200, W=130)
    for op, s in ((OP_FIR, 3.0), (OP_O1, 9.0), (OP_O1, 9.5), (OP_DR, 2.0)):
        R = int(np.ceil((10 if op == OP_DR else 3) * s))
        cuts = [0, 70, 140, 200]
        for k in range(3):
            r0, r1 = cuts[k], cuts[k + 1]
            segs = []
            if r0 > 0:
                segs.append((dev(img[max(0, r0 - R):r0]), max(0, r0 - R)))
            segs.append((dev(img[r0:r1]), r0))
            if r1 < 200:
                segs.append((dev(img[r1:min(200, r1 + R)]), r1))
            outs.append(gc.filter_window(segs, 200, r0, r1 - r0, s, 55.0, 12, op=op))
    # end-to-end host path with several chunks
    os.environ["GC_HOST_CHUNKS"] = "4"
    h = np.ascontiguousarray(config_image("c2", H=300, W=128))
    for op in (OP_FIR, OP_O1, OP_DR):
        outs.append(torch.from_numpy(gc.filter_host(h, 5.0, 70.0, 8, op=op)))
    # guard margins around caller outputs: libgc must write exactly the H x W block
    for op, s in ((OP_FIR, 3.0), (OP_O1, 9.0), (OP_O1, 16.0), (OP_DR, 3.0)):
        x = dev(config_image("c5", H=130, W=98))
        oc = gc.filter(x, s, 55.0, 12, op=op)
        flat = torch.full((130 * 98 + 2 * 4096,), float("nan"), device="cuda")
        mid = flat[4096:4096 + 130 * 98].view(130, 98)            # contiguous block with margins
        gc.filter(x, s, 55.0, 12, op=op, out=mid)
        torch.cuda.synchronize()
        guard_ok = bool(torch.isnan(flat[:4096]).all() and torch.isnan(flat[4096 + 130 * 98:]).all())
        if not guard_ok or not torch.equal(mid, oc):
            print(f"sanitize_cases: guard margin written or result differs (op {op}, sigma_s {s})")
            return 1
    torch.cuda.synchronize()
    bad = [i for i, o in enumerate(outs) if not torch.isfinite(o).all()]
    oob = gc.debug_oob_count() if checked else None
    print(f"sanitize_cases: {len(outs)} calls ({gc.version()}), non-finite outputs: {bad}, "
          f"out-of-bounds accesses: {oob}")
    return 1 if bad or (oob or 0) > 0 else 0


if __name__ == "__main__":
    sys.exit(main())
