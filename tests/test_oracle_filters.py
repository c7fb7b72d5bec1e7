"""Pins for oracle/filters.py against what PAPER.md, SPEC.md examples and
mathematics fix: library routines for special cases (scipy's 'mirror'
correlation = eq. 7), brute force on tiny inputs (mpmath double loops), limits
(sigma_r -> inf, N -> inf), exact identities (constant images, the summation
exchange of P:97), symmetry, and the paper's qualitative Table I ordering.
"""
import json
import math
import os

import mpmath as mp
import numpy as np
import pytest
from scipy import ndimage

import oracle
from synth import checkerboard, config_image, gradient

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_pins.json")))


# ---------------------------------------------------------------- boundary, taps, eq. (7)

def test_mirror_index_examples_and_properties():
    assert oracle.mirror_index(-1, 5) == 1
    assert oracle.mirror_index(5, 5) == 3
    assert oracle.mirror_index(2, 5) == 2
    assert oracle.mirror_index(-7, 1) == 0
    for n in [2, 3, 7]:
        seq = [oracle.mirror_index(p, n) for p in range(-10 * n, 10 * n)]
        assert all(0 <= v < n for v in seq)
        for p in range(-5 * n, 5 * n):           # period 2n-2 and the two reflections
            assert oracle.mirror_index(p, n) == oracle.mirror_index(p + 2 * n - 2, n)
            assert oracle.mirror_index(-p, n) == oracle.mirror_index(p, n)
            assert oracle.mirror_index(n - 1 + p, n) == oracle.mirror_index(n - 1 - p, n)
    # numpy's 'reflect' pad is the same whole-sample extension (single reflection range)
    x = np.arange(9)
    assert list(np.pad(x, 8, mode="reflect")) == [x[oracle.mirror_index(p, 9)] for p in range(-8, 17)]


def test_spatial_taps():
    k, W = oracle.spatial_taps(1.0)
    assert W == 3 and len(k) == 7
    assert k[W] / k[W - 1] == pytest.approx(math.exp(0.5), rel=1e-12)
    assert np.allclose(k, k[::-1]) and k.sum() == pytest.approx(1.0, abs=1e-12)
    assert oracle.spatial_taps(2.5)[1] == 8                        # ceil(3 sigma_s) (R4)
    assert oracle.spatial_taps(16.0)[1] == 48


@pytest.mark.parametrize("shape,sigma_s", [((40, 37), 2.0), ((23, 64), 5.0), ((9, 12), 3.0), ((5, 1), 2.0), ((1, 1), 4.0)])
def test_gauss_fir_equals_scipy_mirror_correlation(shape, sigma_s):
    """Eq. (7) = 2-D correlation with the outer-product kernel, scipy mode='mirror'
    (whole-sample symmetric extension, repeated reflections when W >= n)."""
    rng = np.random.default_rng(7)
    x = rng.uniform(0, 255, size=shape)
    k, W = oracle.spatial_taps(sigma_s)
    ref = ndimage.correlate(x, np.outer(k, k), mode="mirror")
    assert np.max(np.abs(oracle.gauss_fir(x, sigma_s) - ref)) < 1e-10


def test_gauss_fir_impulse_and_constant():
    k, W = oracle.spatial_taps(3.0)
    x = np.zeros((41, 41))
    x[20, 20] = 1.0
    out = oracle.gauss_fir(x, 3.0)
    assert np.allclose(out[20 - W:20 + W + 1, 20 - W:20 + W + 1], np.outer(k, k), atol=1e-16)
    assert out.sum() == pytest.approx(1.0, abs=1e-12)
    assert np.allclose(oracle.gauss_fir(np.full((13, 17), 42.5), 4.0), 42.5, atol=1e-12)


# ---------------------------------------------------------------- eq. (1)

def _direct_mp(f, sigma_s, sigma_r, i, j):
    """Eq. (1) at pixel (i, j) by explicit double loop in 50-digit arithmetic."""
    H, Wd = f.shape
    W = int(math.ceil(3 * sigma_s))
    with mp.workdps(50):
        num = den = mp.mpf(0)
        for a in range(-W, W + 1):
            for b in range(-W, W + 1):
                t = mp.mpf(float(f[oracle.mirror_index(i - a, H), oracle.mirror_index(j - b, Wd)]))
                w = mp.exp(-mp.mpf(a * a + b * b) / (2 * mp.mpf(sigma_s) ** 2)) * \
                    mp.exp(-(t - mp.mpf(float(f[i, j]))) ** 2 / (2 * mp.mpf(sigma_r) ** 2))
                num += w * t
                den += w
        return num / den


def test_direct_filter_brute_force_3x3_checker():
    """3x3 two-level checkerboard, sigma_s=1, sigma_r=30, vs high precision."""
    f = checkerboard(3, 3, 1).astype(np.float64)
    out = oracle.bilateral_direct(f, 1.0, 30.0)
    for i in range(3):
        for j in range(3):
            assert abs(out[i, j] - float(_direct_mp(f, 1.0, 30.0, i, j))) < 1e-9


def test_direct_filter_properties():
    f = config_image("c1", H=24, W=20).astype(np.float64)
    out = oracle.bilateral_direct(f, 2.0, 30.0)
    assert np.allclose(oracle.bilateral_direct(np.full((9, 11), 77.0), 2.0, 30.0), 77.0, atol=1e-10)
    assert np.allclose(oracle.bilateral_direct(f + 13.0, 2.0, 30.0), out + 13.0, atol=1e-9)
    assert np.allclose(oracle.bilateral_direct(f[:, ::-1], 2.0, 30.0), out[:, ::-1], atol=1e-9)
    assert np.allclose(oracle.bilateral_direct(f[::-1], 2.0, 30.0), out[::-1], atol=1e-9)
    W = 6
    ext = np.pad(f, W, mode="reflect")
    lo = ndimage.minimum_filter(ext, size=2 * W + 1)[W:-W, W:-W]
    hi = ndimage.maximum_filter(ext, size=2 * W + 1)[W:-W, W:-W]
    assert np.all(out >= lo - 1e-9) and np.all(out <= hi + 1e-9)
    # sigma_r -> inf: eq. (1) degenerates to the Gaussian filter of eq. (7)
    assert np.max(np.abs(oracle.bilateral_direct(f, 2.0, 1e9) - oracle.gauss_fir(f, 2.0))) < 1e-6
    # random spot checks against the mpmath double loop
    for (i, j) in [(0, 0), (5, 19), (23, 7)]:
        assert abs(out[i, j] - float(_direct_mp(f, 2.0, 30.0, i, j))) < 1e-9


# ---------------------------------------------------------------- GCF

TWIN_CASES = [("c1", 3.0, 100.0, 5), ("c2", 5.0, 70.0, 8), ("c3", 2.0, 60.0, 10), ("c4", 4.0, 85.0, 6),
              ("c5", 3.0, 55.0, 12)]


@pytest.mark.parametrize("cfg,sigma_s,sigma_r,N", TWIN_CASES + [("c2", 3.0, 30.0, 28), ("c1", 2.0, 30.0, 10)])
def test_gc_equals_bruteforce_kernel_sum(cfg, sigma_s, sigma_r, N):
    """Key pin: P/Q of eqs. (6)-(10) equals eq. (1) evaluated with the Gauss-polynomial
    kernel (4) summed directly — the identity the paper derives "by exchanging the
    order of the summations".  Catches a wrong plane index, a dropped
    sigma_r, a wrong centring, a wrong G_n."""
    f = config_image(cfg, H=20, W=23)
    out, nf = oracle.gc_filter(f, sigma_s, sigma_r, N)
    bf, nb = oracle.gc_bruteforce(f, sigma_s, sigma_r, N)
    assert nf == nb            # (sigma_r=30, N=10 is ill-posed on this image: Q <= 0 at some pixels, R1)
    assert np.max(np.abs(out - bf)) < 1e-9


def test_gc_equals_bruteforce_taylor():
    f = config_image("c1", H=18, W=21)
    c = oracle.taylor_c(8)
    out, _ = oracle.gc_filter(f, 3.0, 40.0, 8, c=c)
    bf, _ = oracle.gc_bruteforce(f, 3.0, 40.0, 8, c=c)
    assert np.max(np.abs(out - bf)) < 1e-9


@pytest.mark.parametrize("scheme", ["cheb", "taylor"])
def test_gc_constant_image_fixpoint(scheme):
    """a constant image is returned unchanged (P = sigma_r (g/sigma_r) Q)."""
    for v in [0.0, 37.0, 127.5, 200.0, 255.0]:
        for N in [4, 5, 10]:
            c = None if scheme == "cheb" else oracle.taylor_c(N)
            out, nfb = oracle.gc_filter(np.full((12, 15), v, np.float32), 3.0, 30.0, N, c=c)
            if nfb == 0:
                assert np.max(np.abs(out - v)) < 1e-10
            else:
                assert np.all(out == v)   # guarded pixels pass f through


def test_gc_large_sigma_r_reduces_to_gaussian():
    """sigma_r -> inf: mu -> 0, the range kernel -> 1, output -> eq. (7) applied to f."""
    f = config_image("c2", H=30, W=26).astype(np.float64)
    out, _ = oracle.gc_filter(f, 3.0, 1e6, 6)
    assert np.max(np.abs(out - oracle.gauss_fir(f, 3.0))) < 1e-4


def test_gc_converges_to_direct_filter_as_N_grows():
    """N -> inf at sigma_r=30: the Chebyshev kernel -> exact kernel, GCF -> eq. (1)."""
    f = config_image("c2", H=48, W=48)
    direct = oracle.bilateral_direct(f, 3.0, 30.0)
    errs = []
    for N in [28, 32, 40]:
        out, nf = oracle.gc_filter(f, 3.0, 30.0, N)
        assert nf == 0
        errs.append(oracle.mse_db(out, direct))
    assert errs[0] > errs[1] > errs[2]
    assert errs[2] < -100.0


def test_gc_flip_equivariance():
    f = config_image("c1", H=33, W=29)
    out, _ = oracle.gc_filter(f, 3.0, 100.0, 5)
    assert np.allclose(oracle.gc_filter(f[:, ::-1], 3.0, 100.0, 5)[0], out[:, ::-1], atol=1e-9)
    assert np.allclose(oracle.gc_filter(f[::-1], 3.0, 100.0, 5)[0], out[::-1], atol=1e-9)
    assert np.allclose(oracle.gc_filter(f.T, 3.0, 100.0, 5)[0], out.T, atol=1e-9)


def test_gc_acceptance_ac3():
    """S:469 (AC3): GCF, N=30, sigma_s=3, sigma_r=30 vs eq. (1): <= -40 dB on 64x64
    checkerboard, gradient and constant images (Table I saturates near -40.5 dB)."""
    for img in [checkerboard(64, 64, 8), gradient(64, 64), np.full((64, 64), 100.0, np.float32)]:
        out, _ = oracle.gc_filter(img, 3.0, 30.0, 30)
        assert oracle.mse_db(out, oracle.bilateral_direct(img, 3.0, 30.0)) <= -40.0


def test_table1_ordering_gcf_beats_gpf_on_two_level_image():
    """Table I and Fig. 4 on a synthetic two-level checkerboard
    (S:470): GCF MSE < GPF MSE for every N; at N=10 GCF <= -5 dB and GPF >= +10 dB."""
    pins = GOLD["table1_checker"]
    img = checkerboard(64, 64, 8)
    direct = oracle.bilateral_direct(img, 5.0, 30.0)
    for N in [4, 8, 10, 12, 16, 20]:
        assert N in pins["N"]
        gcf = oracle.mse_db(oracle.gc_filter(img, 5.0, 30.0, N)[0], direct)
        gpf = oracle.mse_db(oracle.gc_filter(img, 5.0, 30.0, N, c=oracle.taylor_c(N))[0], direct)
        assert gcf < gpf, N
        if N == 10:
            assert gcf <= -5.0 and gpf >= 10.0


def test_gc_rows_equals_full():
    f = config_image("c2", H=61, W=40)
    full, _ = oracle.gc_filter(f, 5.0, 70.0, 8)
    rows = [0, 1, 14, 30, 45, 59, 60]
    part, _ = oracle.gc_filter_rows(f, rows, 5.0, 70.0, 8)
    assert np.array_equal(part, full[rows])


def test_gc_tiny_images():
    for shape in [(1, 1), (1, 9), (7, 1), (2, 3)]:
        f = config_image("c1", H=max(shape[0], 2), W=max(shape[1], 2))[:shape[0], :shape[1]]
        out, _ = oracle.gc_filter(f, 3.0, 100.0, 5)
        bf, _ = oracle.gc_bruteforce(f, 3.0, 100.0, 5)
        assert out.shape == shape
        assert np.max(np.abs(out - bf)) < 1e-9
    out, _ = oracle.gc_filter(np.array([[200.0]]), 3.0, 100.0, 5)
    assert abs(out[0, 0] - 200.0) < 1e-10


def test_metrics():
    a = config_image("c1", H=8, W=8)
    assert oracle.mse_db(a, a) == -math.inf
    assert oracle.mse_db(a, a + 1.0) == pytest.approx(0.0, abs=1e-6)
    assert oracle.mse_db(a, a.astype(np.float64) + 10.0) == pytest.approx(20.0, abs=1e-12)
    assert oracle.psnr_db(a, a.astype(np.float64) + 1.0) == pytest.approx(20 * math.log10(255.0))
