"""ORACLE (test infrastructure only) — Chebyshev machinery of PAPER.md §III.

Plain extended-precision (mpmath) transcription of:
  eq. (11) T_l(x) = cos(l arccos x)
  eq. (12) T_{l+1} = 2x T_l - T_{l-1}
  eq. (13) T_l(x) = sum_n a_{l,n} x^n, a via the recursion of (12)
  zeros    xi_k = cos(pi (2k-1) / (2l)), k = 1..l
  eq. (16) + rescaled form after (18): d_l from h(mu xi_k)
  eq. (19) c_n = mu^-n sum_{l=n}^{N} d_l a_{l,n}
  mu = (U-L)^2 / (4 sigma_r^2)
  Taylor c_n = 1/n!

Reading (R2 / SURVEY §8c-Q2): eqs. (16) and (19) are evaluated at
required_dps() decimal digits and rounded once to binary64, because eq. (19)
cancels terms of size ~e^mu down to O(1).
"""
from __future__ import annotations

import math

import mpmath as mp
import numpy as np


def mu_of(sigma_r, L=0.0, U=255.0):
    """mu = (U - L)^2 / (4 sigma_r^2), exact from the binary64 inputs."""
    return mp.mpf(U - L) ** 2 / (4 * mp.mpf(sigma_r) ** 2)


def cheb_T(l, x):
    """T_l(x) = cos(l arccos x), x in [-1, 1]  (eq. 11)."""
    return mp.cos(l * mp.acos(x))


def cheb_T_recurrence(l, x):
    """T_l(x) by T_0 = 1, T_1 = x, T_{l+1} = 2x T_l - T_{l-1}  (eq. 12)."""
    t_prev, t = mp.mpf(1), mp.mpf(x)
    if l == 0:
        return t_prev
    for _ in range(1, l):
        t_prev, t = t, 2 * x * t - t_prev
    return t


def monomial_table(n_max):
    """a[l][n] = coefficient of x^n in T_l(x), 0 <= n <= l <= n_max  (eq. 13).

    Exact Python integers from the recursion that eq. (12) induces:
    a_{0,0} = 1, a_{1,1} = 1, a_{l+1,n} = 2 a_{l,n-1} - a_{l-1,n}.
    """
    a = [[1]]
    if n_max >= 1:
        a.append([0, 1])
    for l in range(1, n_max):
        nxt = [0] * (l + 2)
        for n in range(l + 2):
            up = 2 * a[l][n - 1] if 1 <= n <= l + 1 else 0
            down = a[l - 1][n] if n <= l - 1 else 0
            nxt[n] = up - down
        a.append(nxt)
    return a


def cheb_zeros(l):
    """The l zeros of T_l: xi_k = cos(pi (2k-1) / (2l)), k = 1..l, at the current mp precision."""
    return [mp.cos(mp.pi * (2 * k - 1) / (2 * l)) for k in range(1, l + 1)]


def required_dps(N, mu):
    """Working decimal digits for eqs. (16)/(19) (R2).

    Large mu: eq. (19) cancels terms ~e^mu 2^N down to O(1).  Small mu: eq. (16)
    cancels O(1) samples down to d_l ~ (mu/2)^l / l!, so ~N log10(1/mu) more digits.
    """
    mu = float(mu)
    small = N * max(0.0, math.log10(1.0 / mu)) if mu > 0 else 0.0
    return int(50 + mu / math.log(10) + N * math.log10(2) + small)


def cheb_d(N, mu, dps=None):
    """d_0..d_N of the degree-N expansion of h(x) = exp(x) on [-mu, mu].

    d_0 = (N+1)^-1 sum_k h(mu xi_k);  d_l = 2 (N+1)^-1 sum_k h(mu xi_k) T_l(xi_k),
    xi_k the N+1 zeros of T_{N+1}; T_l(xi_k) evaluated by eq. (11).
    """
    dps = required_dps(N, mu) if dps is None else dps
    with mp.workdps(dps):
        mu = mp.mpf(mu)
        xi = cheb_zeros(N + 1)
        h = [mp.exp(mu * x) for x in xi]
        d = []
        for l in range(N + 1):
            s = mp.fsum(hk * cheb_T(l, xk) for hk, xk in zip(h, xi))
            d.append(s / (N + 1) if l == 0 else 2 * s / (N + 1))
        return d


def cheb_c(N, mu, dps=None):
    """c_0..c_N of eq. (19): c_n = (1/mu)^n sum_{l=n}^{N} d_l a_{l,n}, as mpf."""
    dps = required_dps(N, mu) if dps is None else dps
    a = monomial_table(N)
    with mp.workdps(dps):
        mu = mp.mpf(mu)
        d = cheb_d(N, mu, dps)
        return [mp.fsum(d[l] * a[l][n] for l in range(n, N + 1)) / mu ** n for n in range(N + 1)]


def cheb_c_float(N, sigma_r, L=0.0, U=255.0):
    """Binary64 c_n (rounded once from the extended-precision eq. 19) for sigma_r, [L, U]."""
    mu = mu_of(sigma_r, L, U)
    dps = required_dps(N, mu)
    with mp.workdps(dps):
        return np.array([float(v) for v in cheb_c(N, mu_of(sigma_r, L, U), dps)], dtype=np.float64)


def taylor_c(N):
    """Gauss-polynomial (GPF) coefficients c_n = 1/n!."""
    return np.array([1.0 / math.factorial(n) for n in range(N + 1)], dtype=np.float64)
