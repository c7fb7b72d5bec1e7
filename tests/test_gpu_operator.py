"""GPU tests of the spatial operator of eq. (7) on its own (gc_gaussian) and of
the GCF with the O(1) exact-window operator (GC_OP_O1) against the fp64 oracle.

The oracle's eq. (7) is the separable truncated FIR (oracle.gauss_fir); the O(1) operator
evaluates the same window with a 6-term cosine fit of the taps (max error 1e-6 of the
peak tap, pinned in test_abi.py::test_operator_taps) and fp32 recursions."""
import math

import numpy as np
import pytest

import oracle
from synth import CONFIGS, config_image

pytestmark = pytest.mark.gpu

MAX_ABS, RMS = 1e-2, 1e-3
OP_FIR, OP_O1 = 1, 2


@pytest.fixture(scope="module")
def gc(cuda_device):
    import paper_1605_02178_b200 as gc
    return gc


def _gauss(gc, img, sigma_s, op):
    import torch
    t = torch.from_numpy(np.ascontiguousarray(img, dtype=np.float32)).cuda()
    out = gc.gaussian(t, sigma_s, op=op)
    torch.cuda.synchronize()
    return out.cpu().numpy().astype(np.float64)


@pytest.mark.parametrize("op", [OP_FIR, OP_O1])
@pytest.mark.parametrize("sigma_s", [2.0, 5.0, 16.0])
def test_impulse_response(gc, op, sigma_s):
    """A unit impulse far from the edges returns the outer product of the 1-D taps."""
    W = math.ceil(3 * sigma_s)
    n = 2 * W + 41
    img = np.zeros((n, n + 7), np.float32)
    cy, cx = n // 2, (n + 7) // 2
    img[cy, cx] = 1.0
    out = _gauss(gc, img, sigma_s, op)
    k = gc.operator_taps(sigma_s, op)
    ref = np.zeros_like(out)
    ref[cy - W:cy + W + 1, cx - W:cx + W + 1] = np.outer(k, k)
    assert np.max(np.abs(out - ref)) <= 2e-7 * k.max() ** 2 * 10 + 1e-9
    kx, _ = oracle.spatial_taps(sigma_s)
    ref2 = np.zeros_like(out)
    ref2[cy - W:cy + W + 1, cx - W:cx + W + 1] = np.outer(kx, kx)
    assert np.max(np.abs(out - ref2)) <= 3e-6 * kx.max() ** 2


@pytest.mark.parametrize("op", [OP_FIR, OP_O1])
@pytest.mark.parametrize("sigma_s,H,W", [(1.0, 33, 47), (3.0, 256, 256), (5.0, 131, 300), (10.0, 200, 77),
                                         (16.0, 300, 290), (40.0, 130, 170), (3.0, 1, 50), (4.0, 37, 1),
                                         (12.0, 5, 9)])
def test_gaussian_vs_oracle(gc, op, sigma_s, H, W):
    """eq. (7) of a config-like 0-255 image: GPU vs oracle.gauss_fir (separable fp64 FIR
    with whole-sample mirroring, repeated when W_s >= n)."""
    if op == OP_FIR and math.ceil(3 * sigma_s) > 1024:
        pytest.skip("FIR radius limit")
    img = config_image("c2", H=max(H, 2), W=max(W, 2))[:H, :W]
    out = _gauss(gc, img, sigma_s, op)
    ref = oracle.gauss_fir(img.astype(np.float64), sigma_s)
    tol = 2e-4 if op == OP_FIR else 2e-3
    assert np.max(np.abs(out - ref)) <= tol


@pytest.mark.parametrize("cfg,sigma_s,H,W", [
    ("c1", 3.0, 256, 256),
    ("c2", 5.0, 1024, 1024),
    ("c2", 5.0, 150, 131),
    ("c3", 2.0, 300, 517),
    ("c3", 10.0, 200, 333),
    ("c3", 20.0, 190, 210),
    ("c3", 40.0, 130, 170),
    ("c3", 40.0, 700, 650),
    ("c4", 4.0, 129, 1024),
    ("c5", 6.0, 400, 333),     # W = 18: leaving stream pre-staged, stages first (gc_o1.cu row_o1_task)
    ("c5", 16.0, 300, 290),
    ("c5", 16.0, 1030, 1100),
])
def test_parity_twin_o1(gc, cfg, sigma_s, H, W):
    """GCF with the O(1) operator vs the oracle at the sigma_r twins (R1)."""
    import torch
    c = CONFIGS[cfg]
    img = config_image(c, H=H, W=W)
    t = torch.from_numpy(img).cuda()
    out = gc.filter(t, sigma_s, c.sigma_r_twin, c.N, op=OP_O1)
    torch.cuda.synchronize()
    out = out.cpu().numpy().astype(np.float64)
    ref, nfb = oracle.gc_filter(img, sigma_s, c.sigma_r_twin, c.N)
    assert nfb == 0
    err = np.abs(out - ref)
    ma, rms = float(err.max()), float(math.sqrt(np.mean(err ** 2)))
    assert ma <= MAX_ABS and rms <= RMS, f"{cfg} sigma_s={sigma_s} {H}x{W}: max-abs {ma:.3e} rms {rms:.3e}"


def test_o1_and_fir_agree_on_paper_regime(gc):
    """sigma_r = 30, N = 28 (Table II's operating point): both operators vs the oracle."""
    import torch
    img = config_image("c2", H=160, W=170)
    t = torch.from_numpy(img).cuda()
    ref, _ = oracle.gc_filter(img, 5.0, 30.0, 28)
    for op in [OP_FIR, OP_O1]:
        out = gc.filter(t, 5.0, 30.0, 28, op=op).cpu().numpy().astype(np.float64)
        assert np.max(np.abs(out - ref)) <= MAX_ABS, op


def test_o1_large_degree(gc):
    """N = 40 (21 plane pairs: 4 lanes per column in the O(1) column pass)."""
    import torch
    img = config_image("c2", H=90, W=100)
    t = torch.from_numpy(img).cuda()
    ref, _ = oracle.gc_filter(img, 6.0, 30.0, 40)
    out = gc.filter(t, 6.0, 30.0, 40, op=OP_O1).cpu().numpy().astype(np.float64)
    assert np.max(np.abs(out - ref)) <= MAX_ABS


@pytest.mark.parametrize("op", [OP_FIR, OP_O1])
def test_guard_counts_every_pixel(gc, op):
    """Coefficients with c_0 < 0 and c_n = 0 otherwise give Q = c_0 Fbar_0 < 0 at every pixel:
    the guard of DESIGN.md R8 must pass f through everywhere and count H*W exactly (the
    counter is warp-aggregated in the kernels)."""
    import torch
    img = config_image("c2", H=133, W=257)
    t = torch.from_numpy(img).cuda()
    fb = torch.zeros(1, dtype=torch.int64, device="cuda")
    c = np.zeros(7)
    c[0] = -1.0
    out = gc.filter(t, 5.0, 70.0, 6, c=c, op=op, fallback=fb)
    torch.cuda.synchronize()
    assert int(fb.item()) == img.size
    assert np.array_equal(out.cpu().numpy(), img)


def test_band_path_single_rank_nccl(gc):
    """gc_bilateral_band through a real (one-rank) NCCL communicator: no neighbours, so the
    band is the whole image and must equal gc_filter bit for bit."""
    import os
    import torch
    import torch.distributed as dist
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29531")
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    comm = gc.Comm(0, 1)
    img = config_image("c5", H=300, W=260)
    t = torch.from_numpy(img).cuda()
    for s in [3.0, 16.0]:
        band = gc.bilateral_band(t, 300, 0, s, 55.0, 12, comm)                 # SURVEY 8(b) signature
        full = gc.bilateral_band(t, 300, 0, s, 55.0, 12, comm, op=gc.OP_O1)    # gc_filter_band
        whole = gc.filter(t, s, 55.0, 12)
        comm.wait(timeout_ms=60000)                                             # gc_comm_wait: idle -> OK
        torch.cuda.synchronize()
        assert torch.equal(band, whole)
        if s > 8:
            assert torch.equal(full, whole)                                     # AUTO resolves to O1 here
    with pytest.raises(ValueError):
        gc.bilateral_band(t, 300, 0, 3.0, 55.0, 12, comm, out=torch.empty((299, 260), device="cuda"))
    comm.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("cfg,sigma_s", [("c5", 16.0), ("c3", 40.0)])
def test_parity_full_size_sampled_rows_o1(gc, cfg, sigma_s):
    """The O(1) path at BASELINE's full sizes in bench.py's launch configuration (c5 16384^2,
    c3 4096^2 at sigma_s = 40), twin sigma_r: rows at both edges, at segment-sized strides and
    in the middle, compared with the oracle evaluated at those rows."""
    import torch
    c = CONFIGS[cfg]
    img = config_image(c)
    t = torch.from_numpy(img).cuda()
    out = gc.filter(t, sigma_s, c.sigma_r_twin, c.N)          # GC_OP_AUTO -> O(1) at these radii
    torch.cuda.synchronize()
    H = img.shape[0]
    rows = [0, 1, 47, 48, H // 4 + 3, H // 2, H - 49, H - 2, H - 1]
    o = out[rows].cpu().numpy().astype(np.float64)
    del out, t
    ref, nfb = oracle.gc_filter_rows(img, rows, sigma_s, c.sigma_r_twin, c.N)
    assert nfb == 0
    err = np.abs(o - ref)
    assert err.max() <= MAX_ABS and math.sqrt(np.mean(err ** 2)) <= RMS, (err.max(), math.sqrt(np.mean(err ** 2)))


@pytest.mark.parametrize("op", [OP_FIR, OP_O1])
def test_maximum_degree_and_radius(gc, op):
    """N = GC_N_MAX = 64 (33 plane pairs) and a radius at the FIR limit, W = 1023 (sigma_s = 341),
    the latter on an image far smaller than the window (repeated reflections)."""
    import torch
    img = config_image("c2", H=70, W=90)
    t = torch.from_numpy(img).cuda()
    ref, _ = oracle.gc_filter(img, 4.0, 30.0, 64)
    out = gc.filter(t, 4.0, 30.0, 64, op=op).cpu().numpy().astype(np.float64)
    assert np.max(np.abs(out - ref)) <= MAX_ABS
    s = 341.0                                                   # W_s = 1023
    ref, _ = oracle.gc_filter(img, s, 100.0, 5)
    out = gc.filter(t, s, 100.0, 5, op=op).cpu().numpy().astype(np.float64)
    assert np.max(np.abs(out - ref)) <= MAX_ABS


def test_out_buffer_checks_and_scratch_trim(gc):
    """caller-supplied `out` buffers are checked (shape, dtype, contiguity, device)
    before libgc writes through them; the private scratch pool can be trimmed."""
    import torch
    img = torch.from_numpy(config_image("c2", H=64, W=80)).cuda()
    with pytest.raises(ValueError):
        gc.filter(img, 3.0, 70.0, 8, out=torch.empty((64, 79), device="cuda"))
    with pytest.raises(TypeError):
        gc.filter(img, 3.0, 70.0, 8, out=torch.empty((64, 80), device="cuda", dtype=torch.float16))
    with pytest.raises(TypeError):
        gc.filter(img, 3.0, 70.0, 8, out=torch.empty((80, 64), device="cuda").t())
    with pytest.raises(TypeError):
        gc.filter_host(img.cpu().numpy(), 3.0, 70.0, 8, out=np.empty((64, 40), np.float32))
    with pytest.raises(TypeError):
        gc.filter_host(img.cpu().numpy(), 3.0, 70.0, 8, out=np.empty((64, 80), np.float64))
    a = gc.filter(img, 3.0, 70.0, 8)
    torch.cuda.synchronize()
    gc.scratch_trim(0)
    b = gc.filter(img, 3.0, 70.0, 8)
    torch.cuda.synchronize()
    assert torch.equal(a, b)


# ------------------------------------------------------------------ pair-parallel column pass (k_col_o1p)

@pytest.mark.parametrize("N,sigma_s,H,W", [
    (0, 9.0, 37, 64),      # NP = 1 (one consumer warp)
    (1, 2.0, 40, 62),      # NP = 2, lead-in of 8 (zl = 7: first leaving row inside the last lead-in stage)
    (2, 1.0, 19, 34),      # NP = 2, W_s = 3
    (3, 5.5, 61, 96),      # NP = 3, ragged last fold block
    (4, 3.0, 9, 40),       # NP = 3, image shorter than the lead-in
    (6, 16.0, 131, 98),    # NP = 4
    (8, 12.5, 70, 130),    # NP = 5
    (10, 7.0, 203, 66),    # NP = 6
    (12, 16.0, 97, 160),   # NP = 7 (c5)
    (13, 4.0, 50, 258),    # NP = 8: the largest pair-parallel kernel
    (14, 20.0, 45, 66),    # NP = 8, W_s = 60 > H (repeated mirroring in y)
])
def test_pair_parallel_column_pass(gc, N, sigma_s, H, W):
    """k_col_o1p (even widths, NP <= 8 plane pairs) for every NP, window lengths that are and are
    not multiples of the 4-row stage / NP-row fold block, lead-ins longer than the image: GCF vs
    the oracle (well-conditioned sigma_r = 200)."""
    import torch
    img = config_image("c2", H=H, W=W)
    t = torch.from_numpy(img).cuda()
    out = gc.filter(t, sigma_s, 200.0, N, op=OP_O1)
    torch.cuda.synchronize()
    ref, nfb = oracle.gc_filter(img, sigma_s, 200.0, N)
    err = np.abs(out.cpu().numpy().astype(np.float64) - ref)
    assert nfb == 0
    assert err.max() <= MAX_ABS and math.sqrt(np.mean(err ** 2)) <= RMS, (N, sigma_s, H, W, err.max())


@pytest.mark.parametrize("rows", [(0, 57), (57, 131), (131, 190), (40, 41)])
def test_pair_parallel_column_pass_windows(gc, rows):
    """Interior and edge row windows (gc_filter_window, the band path's building block) through
    k_col_o1p: the producer's per-row boxes at window edges and its clamped entering rows."""
    import torch
    H, W, s = 190, 98, 16.0
    img = config_image("c5", H=H, W=W)
    R = math.ceil(3 * s)
    r0, r1 = rows
    a, b = max(0, r0 - R), min(H, r1 + R)
    seg = torch.from_numpy(np.ascontiguousarray(img[a:b])).cuda()
    out = gc.filter_window([(seg, a)], H, r0, r1 - r0, s, 200.0, 12, op=OP_O1)
    torch.cuda.synchronize()
    ref, _ = oracle.gc_filter_rows(img, list(range(r0, r1)), s, 200.0, 12)
    err = np.abs(out.cpu().numpy().astype(np.float64) - ref)
    assert err.max() <= MAX_ABS and math.sqrt(np.mean(err ** 2)) <= RMS, (rows, err.max())
