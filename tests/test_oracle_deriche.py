"""Pins of oracle/deriche.py (the Deriche-class recursive fast mode):
recursions vs the closed-form kernel they must realise, normalisation, the fit's distance
to the sampled Gaussian (Deriche's own accuracy claim), symmetry, and its documented gap to
eq. (7) inside the GCF."""
import math

import numpy as np
import pytest

import oracle
from oracle import deriche as D
from synth import config_image


@pytest.mark.parametrize("s", [1.0, 2.0, 5.0, 16.0])
def test_recursions_realise_the_closed_form(s):
    """Impulse responses of the causal / anticausal recursions (run on a unit impulse, no
    padding) equal h(k), k >= 0 and h(k), k >= 1 of the closed form (partial fractions)."""
    nc, ma, dd, Z = D.deriche_coeffs(s)
    n = int(40 * s)
    x = np.zeros(n)
    x[0] = 1.0
    yp = np.zeros(n)
    for k in range(n):                                    # causal
        acc = sum(nc[i] * x[k - i] for i in range(4) if k - i >= 0)
        acc -= sum(dd[i - 1] * yp[k - i] for i in range(1, 5) if k - i >= 0)
        yp[k] = acc
    h = D.deriche_kernel(np.arange(n), s)
    assert np.max(np.abs(yp - h)) <= 1e-10                # fp64 recursion over 40 s samples
    xr = np.zeros(n)
    xr[-1] = 1.0
    ym = np.zeros(n)
    for k in range(n - 1, -1, -1):                        # anticausal
        ym[k] = sum(ma[i - 1] * xr[k + i] - dd[i - 1] * ym[k + i] for i in range(1, 5) if k + i < n)
    assert abs(ym[-1]) <= 1e-15                           # h- starts at k = 1
    assert np.max(np.abs(ym[::-1][1:] - h[1:])) <= 1e-10
    # Z = sum over all integers of h(|k|)
    kk = np.arange(-int(60 * s), int(60 * s) + 1)
    assert abs(Z - D.deriche_kernel(kk, s).sum()) <= 1e-9 * Z


@pytest.mark.parametrize("s", [2.0, 5.0, 16.0, 40.0])
def test_fit_is_within_5e4_of_the_sampled_gaussian(s):
    """Deriche's 4th-order fit (P:50's [Deriche1993]) against exp(-m^2/2s^2), both normalised:
    3.2e-4 ... 4.7e-4 of the peak (SURVEY A.5 'Deriche impulse response vs sampled Gaussian')."""
    m = np.arange(-int(15 * s), int(15 * s) + 1)
    h = D.deriche_kernel(m, s)
    h /= h.sum()
    g = np.exp(-m * m / (2 * s * s))
    g /= g.sum()
    rel = np.max(np.abs(h - g)) / g.max()
    assert 2e-4 <= rel <= 5e-4


def test_filter_impulse_constant_symmetry():
    s = 3.0
    n = 400
    x = np.zeros((2, n))
    x[0, 200] = 1.0
    x[1] = 7.5                                            # constant row
    y = D.deriche_filter_1d(x, s)
    k = np.arange(n) - 200
    _, _, _, Z = D.deriche_coeffs(s)
    assert np.max(np.abs(y[0] - D.deriche_kernel(k, s) / Z)) <= 1e-12
    assert np.max(np.abs(y[1] - 7.5)) <= 7.5 * 1e-7       # padding tail beyond 10 s
    rng = np.random.default_rng(0)
    img = rng.uniform(0, 255, (30, 41))
    a = D.deriche_2d(img, 2.5)
    b = D.deriche_2d(img[::-1, ::-1], 2.5)[::-1, ::-1]
    assert np.max(np.abs(a - b)) <= 1e-9


def test_mirror_padding_equals_explicit_extension():
    """The K-sample whole-sample padding is the same extension eq. (7) uses (R5): filtering a
    signal equals filtering its explicit mirror extension and cropping, away from the pad."""
    s = 2.0
    rng = np.random.default_rng(1)
    x = rng.uniform(-1, 1, 37)
    K = D.deriche_pad(s)
    ext = np.array([x[oracle.mirror_index(p, 37)] for p in range(-3 * K, 37 + 3 * K)])
    y = D.deriche_filter_1d(x, s)
    ye = D.deriche_filter_1d(ext, s)[3 * K:3 * K + 37]
    assert np.max(np.abs(y - ye)) <= 1e-6


def test_gcf_gap_to_eq7():
    """The fast mode moves the GCF by a few tenths of a grey level relative to eq. (7)
    (0.24-0.35 max-abs): large enough that it must have its own oracle."""
    img = config_image("c2", H=80, W=90)
    a, _ = oracle.gc_filter(img, 5.0, 70.0, 8)
    b, _ = D.gc_filter_deriche(img, 5.0, 70.0, 8)
    gap = np.max(np.abs(a - b))
    assert 0.02 <= gap <= 1.0
