"""CPU-side checks of libgc.so: it loads, exports every symbol include/gc.h declares,
its host-only entry points (gc_coeffs, gc_band_plan) agree with the oracle / the
paper, and argument validation returns the documented status codes before any CUDA
work is enqueued.  No kernel is launched here."""
import ctypes
import math
import os
import re

import numpy as np
import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def gc():
    import paper_1605_02178_b200 as gc
    if not os.path.exists(gc.LIB_PATH):
        from paper_1605_02178_b200 import build
        build.build()
    return gc


def _declared():
    src = open(os.path.join(ROOT, "include", "gc.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gc_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol(gc):
    lib = gc.lib()
    names = _declared()
    assert "gc_bilateral" in names and "gc_coeffs" in names and "gc_bilateral_batch" in names
    for n in names:
        assert hasattr(lib, n), n
    assert "sm_100a" in gc.version()


def test_library_is_sm100a_only():
    """The fat binary carries sm_100a SASS (cuobjdump), nothing for other archs."""
    import subprocess
    import paper_1605_02178_b200 as gc
    r = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", gc.LIB_PATH], capture_output=True, text=True)
    if r.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    archs = set(re.findall(r"sm_\d+a?", r.stdout))
    assert archs == {"sm_100a"}, archs


STATED = [(5, 30.0), (8, 20.0), (10, 15.0), (6, 25.0), (12, 10.0)]
TWINS = [(5, 100.0), (8, 70.0), (10, 60.0), (6, 85.0), (12, 55.0)]


@pytest.mark.parametrize("N,sigma_r", STATED + TWINS + [(28, 30.0), (40, 30.0), (0, 30.0), (1, 50.0), (20, 1e5)])
def test_gc_coeffs_matches_oracle(gc, N, sigma_r):
    """Step a0: libgc's own multiprecision eq. (19) vs the mpmath oracle (to 1 ulp)."""
    c, mu = gc.coeffs(N, sigma_r)
    ref = oracle.cheb_c_float(N, sigma_r)
    assert mu == float(oracle.mu_of(sigma_r))
    ulps = np.abs(c.view(np.int64) - ref.view(np.int64))
    assert np.all(ulps <= 1), (c, ref)


def test_gc_coeffs_errors(gc):
    lib = gc.lib()
    c = (ctypes.c_double * 80)()
    assert lib.gc_coeffs(-1, 30.0, 0.0, 255.0, c, None) == 1
    assert lib.gc_coeffs(5, 0.0, 0.0, 255.0, c, None) == 1
    assert lib.gc_coeffs(5, 30.0, 255.0, 0.0, c, None) == 1
    assert lib.gc_coeffs(5, float("nan"), 0.0, 255.0, c, None) == 1
    assert lib.gc_coeffs(5, 30.0, 0.0, 255.0, None, None) == 1
    assert lib.gc_coeffs(65, 30.0, 0.0, 255.0, c, None) == 2        # N > GC_N_MAX
    assert lib.gc_coeffs(5, 1.0, 0.0, 255.0, c, None) == 2          # mu = 16256 > GC_MU_MAX
    assert lib.gc_coeffs(5, 30.0, 0.0, 255.0, c, None) == 0


def test_device_entry_points_validate_before_cuda(gc):
    """Bad arguments are rejected with GC_EINVAL / GC_ERANGE without touching CUDA."""
    lib = gc.lib()
    fake = ctypes.c_void_p(0x10000000)
    fake2 = ctypes.c_void_p(0x20000000)
    assert lib.gc_bilateral(None, 8, 8, 3.0, 30.0, 5, fake2, None) == 1
    assert lib.gc_bilateral(fake, 0, 8, 3.0, 30.0, 5, fake2, None) == 1
    assert lib.gc_bilateral(fake, 8, 8, 0.0, 30.0, 5, fake2, None) == 1
    assert lib.gc_bilateral(fake, 8, 8, 3.0, -1.0, 5, fake2, None) == 1
    assert lib.gc_bilateral(fake, 8, 8, 3.0, 30.0, -1, fake2, None) == 1
    assert lib.gc_bilateral(fake, 8, 8, 3.0, 30.0, 65, fake2, None) == 2
    assert lib.gc_bilateral(fake, 8, 8, 3.0, 30.0, 5, fake, None) == 1           # aliased
    assert lib.gc_bilateral_batch(fake, 0, 8, 8, 3.0, 30.0, 5, fake2, None) == 1
    assert lib.gc_bilateral_c(fake, 8, 8, 3.0, 30.0, 5, None, fake2, None) == 1
    cc = (ctypes.c_double * 6)(1, 1, 0.5, float("inf"), 0, 0)
    assert lib.gc_bilateral_c(fake, 8, 8, 3.0, 30.0, 5, cc, fake2, None) == 1
    assert lib.gc_bilateral(fake, 8, 8, 2000.0, 30.0, 5, fake2, None) == 2      # W_s > O(1) limit
    assert lib.gc_gaussian(fake, 1, 8, 8, 2.0, 7, fake2, None) == 1               # unknown operator
    assert lib.gc_gaussian(fake, 1, 8, 8, 500.0, 1, fake2, None) == 2             # W_s > FIR limit
    assert lib.gc_gaussian(fake, 1, 8, 8, 2.0, 1, fake, None) == 1                # aliased
    assert lib.gc_bilateral_direct(None, 1, 8, 8, 2.0, 30.0, fake2, None) == 1
    assert lib.gc_bilateral_direct(fake, 1, 8, 8, 2.0, 0.0, fake2, None) == 1
    assert lib.gc_bilateral_direct(fake, 1, 8, 8, 500.0, 30.0, fake2, None) == 2  # W_s > 1024
    # Deriche operator (GC_OP_DERICHE = 3): N <= 14, fp32 only; validated before CUDA
    p = gc._Params()
    lib.gc_params_init(ctypes.byref(p), 15, 3.0, 30.0)
    p.op = 3
    assert lib.gc_filter(fake, 1, 8, 8, ctypes.byref(p), fake2, None) == 2       # NP = 9 > 8
    p.N, p.precision = 12, 1
    assert lib.gc_filter(fake, 1, 8, 8, ctypes.byref(p), fake2, None) == 1       # binary64 + Deriche
    p.precision, p.op = 0, 4
    assert lib.gc_filter(fake, 1, 8, 8, ctypes.byref(p), fake2, None) == 1       # unknown operator
    assert lib.gc_operator_taps(3.0, 3, None, None) == 1                           # IIR: no finite taps


def test_status_strings(gc):
    lib = gc.lib()
    for s in range(7):
        assert lib.gc_status_string(s).startswith(b"GC_")
    assert lib.gc_status_string(6).startswith(b"GC_ETIMEOUT")


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_band_plan(gc, world):
    H, sigma_s = 1000, 5.0
    R = 15
    rows = [H // world + (1 if k < H % world else 0) for k in range(world)]
    covered = []
    for r in range(world):
        pl = gc.band_plan(H, r, world, rows, sigma_s)
        assert pl["row0"] == sum(rows[:r])
        assert pl["top_rows"] == (R if r > 0 else 0) and pl["top0"] == pl["row0"] - pl["top_rows"]
        assert pl["bot_rows"] == (R if r < world - 1 else 0) and pl["bot0"] == pl["row0"] + rows[r]
        covered += list(range(pl["row0"], pl["row0"] + rows[r]))
    assert covered == list(range(H))


def test_band_plan_errors(gc):
    with pytest.raises(gc.GCError):
        gc.band_plan(100, 0, 2, [50, 49], 3.0)            # rows do not sum to H
    with pytest.raises(gc.GCError):
        gc.band_plan(100, 0, 2, [92, 8], 3.0)             # band <= W_s = 9
    with pytest.raises(gc.GCError):
        gc.band_plan(100, 2, 2, [50, 50], 3.0)            # rank out of range
    gc.band_plan(100, 0, 2, [50, 50], 3.0)                # halo 9 < 50 rows: fine for eq. (7) ...
    with pytest.raises(gc.GCError):
        gc.band_plan(100, 0, 2, [50, 50], 5.0, op=gc.OP_DERICHE)   # ... Deriche needs K = 50 rows: rejected
    with pytest.raises(gc.GCError):
        gc.band_plan(100, 0, 2, [50, 50], 3.0, op=7)      # unknown operator


@pytest.mark.parametrize("world", [1, 2, 3, 8])
@pytest.mark.parametrize("op", [0, 3])
def test_band_exchange_plan(gc, world, op):
    """gc_band_exchange_plan (what gc_filter_band sends, receives and filters): every halo row a
    rank receives is exactly the rows its neighbour sends (offsets into the neighbour's band),
    and the three segments cover [row0 - halo, row0 + H_band + halo) clipped to the image."""
    H, W, sigma_s = 1000, 37, 4.0
    halo = math.ceil((10 if op == 3 else 3) * sigma_s)
    rows = [H // world + (1 if k < H % world else 0) for k in range(world)]
    r0 = [sum(rows[:k]) for k in range(world)]
    plans = [gc.band_exchange_plan(rows[k], W, H, r0[k], k, world, sigma_s, op) for k in range(world)]
    for k, (xf, segs) in enumerate(plans):
        up, down = xf
        assert (up["peer"], down["peer"]) == (k - 1 if k > 0 else -1, k + 1 if k < world - 1 else -1)
        assert segs[1] == (r0[k], rows[k])
        assert segs[0] == (r0[k] - halo, halo if k > 0 else 0)
        assert segs[2] == (r0[k] + rows[k], halo if k < world - 1 else 0)
        for x, seg in ((up, segs[0]), (down, segs[2])):
            if x["peer"] < 0:
                assert x["count"] == 0
                continue
            assert x["count"] == halo * W and x["recv_row0"] == seg[0]
            # what the peer sends to me starts at global row recv_row0
            px = plans[x["peer"]][0][0 if x["peer"] == k + 1 else 1]
            assert px["peer"] == k and px["count"] == x["count"]
            assert r0[x["peer"]] + px["send_offset"] // W == x["recv_row0"] and px["send_offset"] % W == 0


def test_band_exchange_plan_errors(gc):
    with pytest.raises(gc.GCError):
        gc.band_exchange_plan(50, 8, 100, 10, 0, 2, 3.0)     # rank 0 must start at row 0
    with pytest.raises(gc.GCError):
        gc.band_exchange_plan(40, 8, 100, 50, 1, 2, 3.0)     # last rank must end at H
    with pytest.raises(gc.GCError):
        gc.band_exchange_plan(8, 8, 16, 8, 1, 2, 3.0)        # band of 8 rows <= halo 9


@pytest.mark.parametrize("sigma_s", [0.3, 1.0, 2.0, 3.0, 4.0, 5.0, 7.5, 10.0, 16.0, 20.0, 40.0, 100.0, 400.0])
def test_operator_taps(gc, sigma_s):
    """gc_operator_taps: FIR = the sampled, truncated, normalised taps of eq. (7) (oracle
    spatial_taps); the O(1) operator's cosine expansion is within 1e-6 of the peak tap
    on the same window and sums to 1 (a constant plane is preserved)."""
    k, W = oracle.spatial_taps(float(np.float32(sigma_s)))     # the ABI takes sigma_s as fp32
    fir = gc.operator_taps(sigma_s, gc.OP_FIR) if W <= 1024 else None
    o1 = gc.operator_taps(sigma_s, gc.OP_O1)
    assert len(o1) == 2 * W + 1
    if fir is not None:
        assert np.max(np.abs(fir - k)) <= 1e-15
    assert np.max(np.abs(o1 - k)) <= 1e-6 * k.max()
    assert abs(o1.sum() - 1.0) <= 1e-5
    assert np.allclose(o1, o1[::-1], rtol=0, atol=1e-15)            # symmetric (cosines)
    auto = gc.operator_taps(sigma_s, gc.OP_AUTO)
    assert np.array_equal(auto, o1 if W >= 25 else fir)


def test_filter_kernels(gc):
    """gc_filter_kernels (host only): the small-image fused FIR kernel (1 launch) takes FIR calls
    with W_s <= 24 and at most GC_FUSED_MAX_PX = 2^18 output pixels; everything else is 2 passes."""
    if os.environ.get("GC_FIR_FUSED") is not None:
        pytest.skip("GC_FIR_FUSED overrides the dispatch")
    assert gc.filter_kernels(1, 256, 256, 3.0, 40.0, 5) == 1                 # c1: AUTO -> FIR, fused
    assert gc.filter_kernels(1, 512, 512, 5.0, 40.0, 8) == 1                 # 2^18 pixels: still fused
    assert gc.filter_kernels(1, 513, 512, 5.0, 40.0, 8) == 2
    assert gc.filter_kernels(1, 1024, 1024, 5.0, 40.0, 8) == 2               # c2: two passes
    assert gc.filter_kernels(4, 256, 256, 4.0, 40.0, 6) == 1                 # batch counts all images
    assert gc.filter_kernels(5, 256, 256, 4.0, 40.0, 6) == 2
    assert gc.filter_kernels(1, 64, 64, 9.0, 40.0, 5) == 2                   # W = 27: O(1) under AUTO
    assert gc.filter_kernels(1, 64, 64, 9.0, 40.0, 5, op=gc.OP_FIR) == 2     # FIR above W = 24: runtime-W
    assert gc.filter_kernels(1, 64, 64, 3.0, 40.0, 5, op=gc.OP_O1) == 2
    assert gc.filter_kernels(1, 64, 64, 3.0, 40.0, 5, fp64=True) == 2
    with pytest.raises(gc.GCError):
        gc.filter_kernels(0, 64, 64, 3.0, 40.0, 5)
    with pytest.raises(gc.GCError):
        gc.filter_kernels(1, 64, 64, -1.0, 40.0, 5)
