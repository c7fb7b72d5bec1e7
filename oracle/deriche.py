"""ORACLE (test infrastructure only) — the Deriche-class recursive Gaussian "fast mode"
 in binary64.

PAPER.md reaches O(1) cost per pixel for eq. (7) "using separability and recursion" and
cites Deriche's recursive Gaussian for it.  Eq. (7) itself is a truncated
window (R3); this module is the oracle of the *other* reading — the untruncated
4th-order recursive approximation of [Deriche1993] — which the GPU offers as GC_OP_DERICHE.
Its output differs from eq. (7) by ~0.2–0.35 grey levels in the GCF, so it is
checked against this oracle, not against `filters.gauss_fir`.

  deriche_kernel      the closed-form 4th-order fit of Deriche (1993) to the Gaussian:
                      h(x) = (a0 cos(w0 x/s) + a1 sin(w0 x/s)) e^{-b0 x/s}
                           + (c0 cos(w1 x/s) + c1 sin(w1 x/s)) e^{-b1 x/s},  x >= 0, h(-x) = h(x)
  deriche_coeffs      causal / anticausal 4th-order recursions whose impulse responses are
                      h(n), n >= 0 and h(n), n >= 1 (partial fractions of the four poles)
  deriche_filter_1d   y = (y+ + y-) / Z along one axis, Z = sum_n h(n); the signal is padded
                      with K = ceil(10 s) whole-sample mirrored samples per side and the
                      recursions start from zero state (R15)
  deriche_2d          rows, then columns
  gc_filter_deriche   the GCF pipeline of filters.gc_filter with eq. (7)'s operator replaced by
                      deriche_2d
"""
from __future__ import annotations

import math

import numpy as np

from .filters import _gc_combine, _gc_prepare, mirror_index

# Deriche (1993), "Recursively implementing the Gaussian and its derivatives", 4th-order fit
# of exp(-x^2/2) (cited by PAPER P:50 as [Deriche1993]).
DERICHE = dict(a0=1.68, a1=3.735, b0=1.783, b1=1.723, w0=0.6318, w1=1.997, c0=-0.6803, c1=-0.2598)


def deriche_kernel(x, s: float):
    """Closed form h(x) of the 4th-order fit (unnormalised; h(0) = a0 + c0 = 0.9997)."""
    d = DERICHE
    x = np.abs(np.asarray(x, dtype=np.float64)) / s
    return ((d["a0"] * np.cos(d["w0"] * x) + d["a1"] * np.sin(d["w0"] * x)) * np.exp(-d["b0"] * x)
            + (d["c0"] * np.cos(d["w1"] * x) + d["c1"] * np.sin(d["w1"] * x)) * np.exp(-d["b1"] * x))


def _poly_mul(a, b):
    return np.convolve(a, b)


def deriche_coeffs(s: float):
    """(n[0..3], m[1..4], d[1..4], Z) with
         y+[k] = sum_{i=0}^{3} n_i x[k-i] - sum_{i=1}^{4} d_i y+[k-i]     (impulse response h(k), k >= 0)
         y-[k] = sum_{i=1}^{4} m_i x[k+i] - sum_{i=1}^{4} d_i y-[k+i]     (impulse response h(k), k >= 1)
       and Z = sum_{k in Z} h(|k|), from h(k) = sum_j r_j q_j^k (four complex poles q_j)."""
    d = DERICHE
    r = [(d["a0"] - 1j * d["a1"]) / 2, (d["a0"] + 1j * d["a1"]) / 2,
         (d["c0"] - 1j * d["c1"]) / 2, (d["c0"] + 1j * d["c1"]) / 2]
    q = [np.exp((-d["b0"] + 1j * d["w0"]) / s), np.exp((-d["b0"] - 1j * d["w0"]) / s),
         np.exp((-d["b1"] + 1j * d["w1"]) / s), np.exp((-d["b1"] - 1j * d["w1"]) / s)]
    # D(u) = prod_j (1 - q_j u): the same polynomial serves z^{-1} (causal) and z (anticausal)
    D = np.array([1.0 + 0j])
    for qj in q:
        D = _poly_mul(D, [1.0, -qj])
    # causal numerator: sum_j r_j prod_{l != j} (1 - q_l u)
    Nc = np.zeros(4, dtype=complex)
    for j in range(4):
        t = np.array([1.0 + 0j])
        for l in range(4):
            if l != j:
                t = _poly_mul(t, [1.0, -q[l]])
        Nc += r[j] * t
    # anticausal: H-(z) = sum_j r_j (1/(1 - q_j z) - 1) = (Nc(z) - (sum_j r_j) D(z)) / D(z)
    Na = np.concatenate([Nc, [0]]) - sum(r) * D
    assert abs(Na[0]) < 1e-12
    Z = (Nc.sum() / D.sum()).real + (Na.sum() / D.sum()).real     # H+(1) + H-(1)
    return Nc.real.copy(), Na[1:].real.copy(), D[1:].real.copy(), float(Z)


def deriche_pad(s: float) -> int:
    """Mirror padding per side, K = ceil(10 s): the recursions' tails beyond it are < 4e-8."""
    return int(math.ceil(10.0 * s))


def deriche_filter_1d(x: np.ndarray, s: float, axis: int = -1) -> np.ndarray:
    """(y+ + y-) / Z along `axis` with K mirrored samples per side and zero initial state."""
    x = np.moveaxis(np.asarray(x, dtype=np.float64), axis, -1)
    n = x.shape[-1]
    K = deriche_pad(s)
    idx = np.array([mirror_index(p, n) for p in range(-K, n + K)])
    xp = x[..., idx]
    L = xp.shape[-1]
    nc, ma, dd, Z = deriche_coeffs(s)
    yp = np.zeros_like(xp)
    for k in range(L):                                  # causal, left to right
        acc = nc[0] * xp[..., k]
        for i in range(1, 4):
            if k - i >= 0:
                acc = acc + nc[i] * xp[..., k - i]
        for i in range(1, 5):
            if k - i >= 0:
                acc = acc - dd[i - 1] * yp[..., k - i]
        yp[..., k] = acc
    ym = np.zeros_like(xp)
    for k in range(L - 1, -1, -1):                      # anticausal, right to left
        acc = np.zeros_like(xp[..., k])
        for i in range(1, 5):
            if k + i < L:
                acc = acc + ma[i - 1] * xp[..., k + i] - dd[i - 1] * ym[..., k + i]
        ym[..., k] = acc
    y = (yp + ym)[..., K:K + n] / Z
    return np.moveaxis(y, -1, axis)


def deriche_2d(img: np.ndarray, s: float) -> np.ndarray:
    """The separable fast-mode operator: rows (x), then columns (y)."""
    return deriche_filter_1d(deriche_filter_1d(img, s, axis=1), s, axis=0)


def gc_filter_deriche(f, sigma_s, sigma_r, N, c=None, L=0.0, U=255.0):
    """GCF with the N+2 filterings done by deriche_2d instead of eq. (7)."""
    f, g, tc, c = _gc_prepare(f, sigma_r, N, c, L, U)
    e = np.exp(-(g * g) / (2.0 * sigma_r * sigma_r))
    F = [e * (g / sigma_r) ** n for n in range(N + 2)]
    Fbar = [deriche_2d(Fn, sigma_s) for Fn in F]
    return _gc_combine(f, g, Fbar, c, sigma_r, N, tc)
