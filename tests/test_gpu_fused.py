"""The small-image FIR path (csrc/gc_fused.cu) against the two-pass FIR path and the oracle.

The library picks the fused kernel for FIR calls of at most kFuMaxPx output pixels; the
environment variable GC_FIR_FUSED=0 / 1 forces either path (read once per process), so each
side runs in its own subprocess on the same seeded inputs.  The fused kernel performs the
two-pass path's arithmetic operation by operation, hence the comparison is bit for bit
(outputs and guard counts); each case is also gated against the fp64 oracle.
"""
import json
import math
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
from synth import voronoi_texture

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (B, H, W, sigma_s, sigma_r, N, kind): kind "gcf" = gc.filter (op FIR), "raw" = gc.gaussian (op FIR),
# "win" = gc.filter_window on a middle band of rows
CASES = [                                        # sigma_r: the configs' parity twins (synth CONFIGS)
    (1, 1, 1, 3.0, 100.0, 5, "gcf"),
    (1, 1, 77, 3.0, 100.0, 5, "gcf"),
    (1, 77, 1, 3.0, 100.0, 5, "gcf"),
    (1, 256, 256, 3.0, 100.0, 5, "gcf"),         # c1 shape
    (1, 77, 301, 3.0, 100.0, 5, "gcf"),          # ragged tiles in x and y
    (1, 150, 131, 5.0, 70.0, 8, "gcf"),          # c2 operator, odd width
    (3, 65, 97, 4.0, 85.0, 6, "gcf"),            # batch, c4 operator
    (1, 20, 30, 8.0, 60.0, 10, "gcf"),           # W = 24 > image: repeated reflections
    (1, 300, 200, 1.0, 120.0, 3, "gcf"),         # W = 3
    (1, 129, 160, 5.0, 8.0, 8, "gcf"),           # small sigma_r: the guard fires
    (2, 70, 90, 5.0, 0.0, 0, "raw"),             # eq. (7) alone
    (1, 200, 180, 5.0, 70.0, 8, "win"),          # row window (band) of 60 rows at row 70
]

WORKER = r"""
import json, sys
import numpy as np, torch
import paper_1605_02178_b200 as gc
sys.path.insert(0, {root!r})
from synth import voronoi_texture
cases = json.loads(sys.argv[1]); out_path = sys.argv[2]
res = {{}}
for k, (B, H, W, s, sr, N, kind) in enumerate(cases):
    img = np.stack([voronoi_texture(H, W, 100 + 7 * k + b, 24, 10.0) for b in range(B)]).astype(np.float32)
    t = torch.from_numpy(img).cuda()
    fb = torch.zeros(1, dtype=torch.int64, device="cuda")
    if kind == "gcf":
        o = gc.filter(t if B > 1 else t[0], s, sr, N, op=gc.OP_FIR, fallback=fb)
    elif kind == "raw":
        o = gc.gaussian(t, s, op=gc.OP_FIR)
    else:
        o = gc.filter_window([(t[0], 0)], H, 70, 60, s, sr, N, op=gc.OP_FIR)
    torch.cuda.synchronize()
    res[f"o{{k}}"] = o.cpu().numpy()
    res[f"g{{k}}"] = np.array([fb.item()])
np.savez(out_path, **res)
"""


def _run(tmp_path, fused):
    path = str(tmp_path / f"fused{fused}.npz")
    env = dict(os.environ, GC_FIR_FUSED=str(fused), PYTHONPATH=ROOT)
    r = subprocess.run([sys.executable, "-c", WORKER.format(root=ROOT), json.dumps(CASES), path],
                       env=env, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return np.load(path)


@pytest.fixture(scope="module")
def both(tmp_path_factory, cuda_device):
    d = tmp_path_factory.mktemp("fused")
    return _run(d, 1), _run(d, 0)


@pytest.mark.parametrize("k", range(len(CASES)))
def test_fused_equals_two_pass(both, k):
    fu, tp = both
    a, b = fu[f"o{k}"], tp[f"o{k}"]
    assert a.shape == b.shape
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32)), \
        f"case {CASES[k]}: max diff {np.abs(a.astype(np.float64) - b).max():.3e}"
    assert int(fu[f"g{k}"][0]) == int(tp[f"g{k}"][0])


@pytest.mark.parametrize("k", [3, 4, 6, 7, 10, 11])
def test_fused_vs_oracle(both, k):
    fu, _ = both
    B, H, W, s, sr, N, kind = CASES[k]
    out = fu[f"o{k}"].astype(np.float64).reshape(B, -1, W)
    for b in range(B):
        img = voronoi_texture(H, W, 100 + 7 * k + b, 24, 10.0).astype(np.float64)
        if kind == "raw":
            ref = oracle.gauss_fir(img, s)
        elif kind == "win":
            ref = oracle.gc_filter(img, s, sr, N)[0][70:130]
        else:
            ref = oracle.gc_filter(img, s, sr, N)[0]
        err = np.abs(out[b] - ref)
        ma, rms = float(err.max()), float(math.sqrt(np.mean(err ** 2)))
        assert ma <= 1e-2 and rms <= 1e-3, f"case {CASES[k]} image {b}: max-abs {ma:.3e} rms {rms:.3e}"
