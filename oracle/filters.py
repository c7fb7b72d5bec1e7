"""ORACLE (test infrastructure only) — the filters of PAPER.md §I-§III in binary64.

Plain numpy transcription, vectorised over pixels only (loops over window
offsets and polynomial terms are explicit, in the paper's order):

  mirror_index      symmetric extension of f outside I; whole-sample
                    reflection (R5 / SURVEY §8c-Q5)
  spatial_taps      g_{sigma_s} on Omega = [-W, W], W = ceil(3 sigma_s) (
                    DESIGN.md R4), normalised (cancels in eqs. 1 and 10; R6)
  gauss_fir         eq. (7) F_bar(i) = sum_{j in Omega} g_{sigma_s}(j) F(i-j),
                    evaluated separably (rows, then columns) — the 2-D Gaussian is the
                    outer product of the 1-D taps
  bilateral_direct  eq. (1), the direct O(sigma_s^2) filter
  gc_filter         GCF pipeline: centre (eq. 17), auxiliary images (eq. 6),
                    N+2 filterings (eq. 7), P and Q (eqs. 8, 9), ratio (eq. 10),
                    uncentre; Q guard per DESIGN.md R8
  gc_filter_rows    the same, evaluated only at the requested output rows
  gc_bruteforce     eq. (1) with the range kernel replaced by the Gauss-polynomial kernel
                    of eq. (4), summed directly — the sum that eqs. (5)-(10)
                    rearrange "by exchanging the order of the summations"
  mse_db            10 log10(MSE)
"""
from __future__ import annotations

import math

import numpy as np

from .chebyshev import cheb_c_float


# ---------------------------------------------------------------- boundary and taps

def mirror_index(p: int, n: int) -> int:
    """Whole-sample symmetric extension: x(-p) = x(p), x(n-1+p) = x(n-1-p)  (R5).

    Reflection repeats until the index is in [0, n-1] (period 2n-2); n = 1 -> 0.
    """
    if n == 1:
        return 0
    while p < 0 or p > n - 1:
        if p < 0:
            p = -p
        if p > n - 1:
            p = 2 * (n - 1) - p
    return p


def _mirror_range(n: int, W: int) -> np.ndarray:
    """Indices mirror_index(p, n) for p = -W .. n-1+W."""
    return np.array([mirror_index(p, n) for p in range(-W, n + W)], dtype=np.int64)


def spatial_taps(sigma_s: float):
    """(taps, W): taps[m + W] = exp(-m^2 / (2 sigma_s^2)) / sum, |m| <= W = ceil(3 sigma_s)."""
    W = int(math.ceil(3.0 * sigma_s))
    m = np.arange(-W, W + 1, dtype=np.float64)
    k = np.exp(-(m * m) / (2.0 * sigma_s * sigma_s))
    return k / k.sum(), W


# ---------------------------------------------------------------- eq. (7)

def gauss_fir(img: np.ndarray, sigma_s: float) -> np.ndarray:
    """Eq. (7) on a whole image: horizontal pass, then vertical pass, mirror boundary."""
    x = np.asarray(img, dtype=np.float64)
    k, W = spatial_taps(sigma_s)
    H, Wd = x.shape
    ext = x[:, _mirror_range(Wd, W)]                      # ext[:, W + c] = x(:, c)
    tmp = np.zeros((H, Wd))
    for m in range(-W, W + 1):                            # sum_m k[m] x(i - m)
        tmp += k[m + W] * ext[:, W - m: W - m + Wd]
    ext = tmp[_mirror_range(H, W), :]
    out = np.zeros((H, Wd))
    for m in range(-W, W + 1):
        out += k[m + W] * ext[W - m: W - m + H, :]
    return out


# ---------------------------------------------------------------- eq. (1)

def bilateral_direct(f: np.ndarray, sigma_s: float, sigma_r: float) -> np.ndarray:
    """Eq. (1): B[f](i) = sum_j gs(j) gr(f(i-j)-f(i)) f(i-j) / sum_j gs(j) gr(f(i-j)-f(i)).

    Omega = [-W, W]^2, W = ceil(3 sigma_s), row-major offset order, mirror boundary.
    """
    f = np.asarray(f, dtype=np.float64)
    H, Wd = f.shape
    W = int(math.ceil(3.0 * sigma_s))
    ext = f[_mirror_range(H, W)][:, _mirror_range(Wd, W)]
    num = np.zeros((H, Wd))
    den = np.zeros((H, Wd))
    for jy in range(-W, W + 1):
        for jx in range(-W, W + 1):
            gs = math.exp(-(jy * jy + jx * jx) / (2.0 * sigma_s * sigma_s))
            t = ext[W - jy: W - jy + H, W - jx: W - jx + Wd]          # f(i - j)
            w = gs * np.exp(-((t - f) ** 2) / (2.0 * sigma_r * sigma_r))
            num += w * t
            den += w
    return num / den


# ---------------------------------------------------------------- GCF (eqs. 6-10, 17)

def _gc_prepare(f, sigma_r, N, c, L, U):
    f = np.clip(np.asarray(f, dtype=np.float64), L, U)        # R7: inputs clamped to [L, U]
    tc = 0.5 * (L + U)                                         # t_c = (L+U)/2
    g = f - tc                                                 # eq. (17)
    if c is None:
        c = cheb_c_float(N, sigma_r, L, U)                     # eq. (19)
    c = np.asarray(c, dtype=np.float64)
    if c.shape != (N + 1,):
        raise ValueError("need N+1 coefficients")
    return f, g, tc, c


def _gc_combine(f_at, g_at, Fbar, c, sigma_r, N, tc):
    G = [(g_at / sigma_r) ** n for n in range(N + 1)]          # eq. (6) G_n at the output pixels
    P = sigma_r * sum(c[n] * G[n] * Fbar[n + 1] for n in range(N + 1))   # eq. (8)
    Q = sum(c[n] * G[n] * Fbar[n] for n in range(N + 1))                 # eq. (9)
    ok = np.isfinite(P) & np.isfinite(Q) & (Q > 0)                       # R8 guard
    with np.errstate(divide="ignore", invalid="ignore"):
        out = np.where(ok, P / Q + tc, f_at)                             # eq. (10) + uncentre
    return out, int((~ok).sum())


def gc_filter(f, sigma_s, sigma_r, N, c=None, L=0.0, U=255.0):
    """GCF on the whole image.  Returns (output, number of guarded pixels).

    c=None -> Chebyshev c_n of eq. (19); pass taylor_c(N) for the GPF of [Chaudhury2015].
    """
    f, g, tc, c = _gc_prepare(f, sigma_r, N, c, L, U)
    e = np.exp(-(g * g) / (2.0 * sigma_r * sigma_r))
    F = [e * (g / sigma_r) ** n for n in range(N + 2)]                   # eq. (6), n = 0..N+1
    Fbar = [gauss_fir(Fn, sigma_s) for Fn in F]                          # eq. (7), N+2 filterings
    return _gc_combine(f, g, Fbar, c, sigma_r, N, tc)


def gc_filter_rows(f, rows, sigma_s, sigma_r, N, c=None, L=0.0, U=255.0):
    """GCF evaluated only at output rows `rows` (for sampled parity on large images)."""
    rows = np.asarray(rows, dtype=np.int64)
    H = np.asarray(f).shape[0]
    W = int(math.ceil(3.0 * sigma_s))
    need = sorted({mirror_index(int(r) + m, H) for r in rows for m in range(-W, W + 1)})
    sub = np.asarray(f)[need]
    fs, gs, tc, c = _gc_prepare(sub, sigma_r, N, c, L, U)
    e = np.exp(-(gs * gs) / (2.0 * sigma_r * sigma_r))
    # Scatter the needed rows back into an image-shaped view by index map so that
    # the mirrored vertical window below reads exactly the same rows as gc_filter.
    pos = {r: i for i, r in enumerate(need)}
    Fbar = []
    for n in range(N + 2):
        Fn_sub = e * (gs / sigma_r) ** n
        Fbar.append(_fir_rows_from_subset(Fn_sub, pos, H, rows, sigma_s))
    f_at = fs[[pos[int(r)] for r in rows]]
    g_at = gs[[pos[int(r)] for r in rows]]
    return _gc_combine(f_at, g_at, Fbar, c, sigma_r, N, tc)


def _fir_rows_from_subset(sub, pos, H, rows, sigma_s):
    """Eq. (7) at output rows `rows`: horizontal pass on every stored row, then the
    vertical sum over the mirrored rows r - m (same separable sums as gauss_fir)."""
    k, W = spatial_taps(sigma_s)
    Wd = sub.shape[1]
    ext = sub[:, _mirror_range(Wd, W)]
    hsub = np.zeros(sub.shape)
    for q in range(-W, W + 1):
        hsub += k[q + W] * ext[:, W - q: W - q + Wd]
    out = np.zeros((len(rows), Wd))
    for m in range(-W, W + 1):
        src = [pos[mirror_index(int(r) - m, H)] for r in rows]
        out += k[m + W] * hsub[src]
    return out


def gc_bruteforce(f, sigma_s, sigma_r, N, c=None, L=0.0, U=255.0):
    """Eq. (1) with g_{sigma_r}(t - tau) replaced by the Gauss-polynomial kernel (4):

        K(tau, t) = exp(-tau^2/2sr^2) exp(-t^2/2sr^2) sum_n c_n (tau t / sr^2)^n,
        tau = g(i), t = g(i-j)  (centred, eq. 17),

    summed directly over Omega (no auxiliary images).  Equal to gc_filter up to
    rounding by the rearrangement of P:97; guard as in gc_filter.
    """
    f, g, tc, c = _gc_prepare(f, sigma_r, N, c, L, U)
    H, Wd = f.shape
    k, W = spatial_taps(sigma_s)
    rr = _mirror_range(H, W)
    cc = _mirror_range(Wd, W)
    gext = g[rr][:, cc]
    num = np.zeros((H, Wd))
    den = np.zeros((H, Wd))
    s2 = sigma_r * sigma_r
    for jy in range(-W, W + 1):
        for jx in range(-W, W + 1):
            t = gext[W - jy: W - jy + H, W - jx: W - jx + Wd]
            x = g * t / s2
            poly = sum(c[n] * x ** n for n in range(N + 1))
            K = np.exp(-(g * g) / (2 * s2)) * np.exp(-(t * t) / (2 * s2)) * poly
            w = k[jy + W] * k[jx + W] * K
            num += w * (t + tc)                               # f(i-j) = g(i-j) + t_c
            den += w
    ok = np.isfinite(num) & np.isfinite(den) & (den > 0)
    with np.errstate(divide="ignore", invalid="ignore"):
        out = np.where(ok, num / den, f)
    return out, int((~ok).sum())


# ---------------------------------------------------------------- metrics

def mse_db(a, b) -> float:
    """10 log10(|I|^-1 sum (a - b)^2); -inf for identical images."""
    d = np.asarray(a, dtype=np.float64) - np.asarray(b, dtype=np.float64)
    m = float(np.mean(d * d))
    return -math.inf if m == 0.0 else 10.0 * math.log10(m)


def psnr_db(a, b, peak=255.0) -> float:
    return 10.0 * math.log10(peak * peak) - mse_db(a, b)


def max_abs(a, b) -> float:
    return float(np.max(np.abs(np.asarray(a, dtype=np.float64) - np.asarray(b, dtype=np.float64))))


def rms(a, b) -> float:
    d = np.asarray(a, dtype=np.float64) - np.asarray(b, dtype=np.float64)
    return float(math.sqrt(np.mean(d * d)))
