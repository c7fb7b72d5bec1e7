"""GPU direct bilateral filter of eq. (1) (gc_bilateral_direct) against
the fp64 oracle (oracle.bilateral_direct), element by element."""
import numpy as np
import pytest

import oracle
from synth import config_image

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gc(cuda_device):
    import paper_1605_02178_b200 as gc
    return gc


def _direct(gc, img, sigma_s, sigma_r):
    import torch
    t = torch.from_numpy(np.ascontiguousarray(img, dtype=np.float32)).cuda()
    out = gc.bilateral_direct(t, sigma_s, sigma_r)
    torch.cuda.synchronize()
    return out.cpu().numpy().astype(np.float64)


@pytest.mark.parametrize("cfg,sigma_s,sigma_r,H,W", [
    ("c1", 3.0, 30.0, 64, 80), ("c2", 5.0, 20.0, 70, 61), ("c3", 2.0, 15.0, 40, 100),
    ("c4", 4.0, 25.0, 33, 47), ("c5", 6.0, 10.0, 50, 45), ("c2", 12.0, 30.0, 17, 23),   # W_s >= n
    ("c1", 1.0, 100.0, 1, 9), ("c1", 2.0, 50.0, 7, 1), ("c1", 3.0, 30.0, 1, 1),
])
def test_direct_vs_oracle(gc, cfg, sigma_s, sigma_r, H, W):
    img = config_image(cfg, H=max(H, 2), W=max(W, 2))[:H, :W]
    out = _direct(gc, img, sigma_s, sigma_r)
    ref = oracle.bilateral_direct(img.astype(np.float64), sigma_s, sigma_r)
    assert np.max(np.abs(out - ref)) <= 2e-3


def test_direct_constant_and_batch(gc):
    import torch
    img = np.full((20, 30), 77.0, np.float32)
    assert np.max(np.abs(_direct(gc, img, 3.0, 10.0) - 77.0)) <= 1e-4
    imgs = np.stack([config_image("c4", index=i, H=40, W=50) for i in range(3)])
    t = torch.from_numpy(imgs).cuda()
    ob = gc.bilateral_direct(t, 4.0, 25.0)
    for i in range(3):
        assert torch.equal(ob[i], gc.bilateral_direct(t[i].contiguous(), 4.0, 25.0))
