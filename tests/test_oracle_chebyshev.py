"""Pins for oracle/chebyshev.py against what PAPER.md and mathematics fix.

None of these re-types the oracle's own formula: each compares against a
printed value, a closed form (binomial formula, Bessel-function aliasing
identity), an independent route to the same unique object (Vandermonde
solve), a limit, or an error bound.
"""
import json
import math
import os

import mpmath as mp
import numpy as np
import pytest

import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_pins.json")))

# (N, sigma_r): the five stated BASELINE configs, their sigma_r twins, the paper's regime
STATED = [(5, 30.0), (8, 20.0), (10, 15.0), (6, 25.0), (12, 10.0)]
TWINS = [(5, 100.0), (8, 70.0), (10, 60.0), (6, 85.0), (12, 55.0)]
PAPER = [(10, 30.0), (20, 30.0), (28, 30.0)]


def test_low_order_rows_printed_in_paper():
    a = oracle.monomial_table(4)
    for l, row in GOLD["chebyshev_low_order"]["monomial_rows"].items():
        assert a[int(l)] == row
    assert a[4] == GOLD["chebyshev_row4"]["row"]


def test_monomial_table_closed_form():
    """a_{l,l-2k} = (-1)^k 2^{l-2k-1} l/(l-k) C(l-k,k) (l>=1), zero for odd l-n."""
    a = oracle.monomial_table(64)
    assert a[0] == [1]
    for l in range(1, 65):
        for n in range(l + 1):
            if (l - n) % 2:
                assert a[l][n] == 0
                continue
            k = (l - n) // 2
            num = (-1) ** k * l * math.comb(l - k, k) * 2 ** (l - 2 * k)
            assert num % (2 * (l - k)) == 0
            assert a[l][n] == num // (2 * (l - k)), (l, n)


def test_monomial_table_matches_trig_definition():
    """Eq. (13) evaluated vs eq. (11) cos(l arccos x), and eq. (12) vs eq. (11)."""
    a = oracle.monomial_table(40)
    with mp.workdps(60):
        for x in [mp.mpf(-1), mp.mpf("-0.73"), mp.mpf("0.1"), mp.mpf("0.5"), mp.mpf("0.999"), mp.mpf(1)]:
            for l in range(41):
                poly = mp.fsum(a[l][n] * x ** n for n in range(l + 1))
                ref = mp.cos(l * mp.acos(x))
                assert abs(poly - ref) < mp.mpf(10) ** -40
                assert abs(oracle.cheb_T_recurrence(l, x) - ref) < mp.mpf(10) ** -40
        # printed example T_2(0.5) = -0.5 (SPEC S:237 from P:130)
        assert oracle.cheb_T(2, mp.mpf("0.5")) == pytest.approx(-0.5, abs=1e-50)


def test_zeros_are_zeros_of_T():
    """xi_k are l distinct roots in (-1, 1) of the eq.-(13) polynomial T_l."""
    a = oracle.monomial_table(33)
    with mp.workdps(50):
        for l in [1, 2, 3, 6, 9, 13, 33]:
            xi = oracle.cheb_zeros(l)
            assert len(xi) == l
            assert all(-1 < x < 1 for x in xi)
            assert all(xi[i] > xi[i + 1] for i in range(l - 1))
            for x in xi:
                assert abs(mp.fsum(a[l][n] * x ** n for n in range(l + 1))) < mp.mpf(10) ** -35
        assert oracle.cheb_zeros(1)[0] == pytest.approx(0.0, abs=1e-40)
        z3 = oracle.cheb_zeros(3)
        assert float(z3[0]) == pytest.approx(math.sqrt(3) / 2, abs=1e-15)


def test_discrete_orthogonality_eq14():
    a = oracle.monomial_table(20)
    with mp.workdps(40):
        for l in [1, 2, 5, 11, 20]:
            xi = oracle.cheb_zeros(l)
            T = [[mp.fsum(a[i][n] * x ** n for n in range(i + 1)) for x in xi] for i in range(l)]
            for i in range(l):
                for j in range(l):
                    s = mp.fsum(T[i][k] * T[j][k] for k in range(l))
                    want = 0 if i != j else (l if i == 0 else mp.mpf(l) / 2)
                    assert abs(s - want) < mp.mpf(10) ** -30, (l, i, j)


@pytest.mark.parametrize("N,sigma_r", STATED + TWINS + PAPER)
def test_mu(N, sigma_r):
    for L, U, s, want in GOLD["mu_examples"]["cases"]:
        assert float(oracle.mu_of(s, L, U)) == want
    with mp.workdps(50):
        assert oracle.mu_of(sigma_r) * 4 * mp.mpf(sigma_r) ** 2 == 255 ** 2


def _bessel_d(N, mu, dps):
    """Chebyshev-node coefficients of e^{mu x} from the modified Bessel expansion
    e^{mu x} = I_0(mu) + 2 sum I_m(mu) T_m(x) and the aliasing of T_m at the zeros of
    T_{N+1}: T_{2q(N+1) +- l}(xi_k) = (-1)^q T_l(xi_k)."""
    with mp.workdps(dps):
        d = []
        for l in range(N + 1):
            s = mp.besseli(l, mu)
            q = 1
            while True:
                t1 = mp.besseli(2 * q * (N + 1) - l, mu)
                t2 = mp.besseli(2 * q * (N + 1) + l, mu)  # l = 0: both aliases are m = 2q(N+1)
                s += (-1) ** q * (t1 + t2)
                if abs(t1) < mp.mpf(10) ** (-dps) * abs(s):
                    break
                q += 1
            d.append(s if l == 0 else 2 * s)
        return d


@pytest.mark.parametrize("N,sigma_r", STATED + TWINS + PAPER + [(10, 127.5)])
def test_d_matches_bessel_aliasing_identity(N, sigma_r):
    dps = oracle.required_dps(N, oracle.mu_of(sigma_r))
    with mp.workdps(dps):
        mu = oracle.mu_of(sigma_r)
        d = oracle.cheb_d(N, mu, dps)
        ref = _bessel_d(N, mu, dps)
        for l in range(N + 1):
            assert abs(d[l] - ref[l]) <= mp.mpf(10) ** (-25) * abs(ref[l]), l


def test_d_worked_example_mu1():
    """N=10, mu=1: d_l -> 2 I_l(1) (I_0 for l=0) to within the aliasing residue."""
    d = oracle.cheb_d(10, 1)
    for l in range(7):
        ref = mp.besseli(l, 1) * (1 if l == 0 else 2)
        assert abs(float(d[l]) - float(ref)) < 1e-14


@pytest.mark.parametrize("N,sigma_r", STATED + TWINS + PAPER)
def test_c_interpolates_exp_at_nodes(N, sigma_r):
    """sum_n c_n (mu xi_k)^n = exp(mu xi_k): eq. (19) represents the interpolant of eq. (16)."""
    dps = oracle.required_dps(N, oracle.mu_of(sigma_r))
    with mp.workdps(dps):
        mu = oracle.mu_of(sigma_r)
        c = oracle.cheb_c(N, mu, dps)
        for x in oracle.cheb_zeros(N + 1):
            p = mp.fsum(c[n] * (mu * x) ** n for n in range(N + 1))
            assert abs(p - mp.exp(mu * x)) < mp.mpf(10) ** -30 * mp.exp(mu)  # cancellation scale e^mu


@pytest.mark.parametrize("N,sigma_r", STATED + TWINS + [(10, 30.0), (28, 30.0)])
def test_c_equals_vandermonde_solve(N, sigma_r):
    """The degree-N interpolant through the N+1 nodes is unique: solve V c = e^{nodes} directly."""
    dps = oracle.required_dps(N, oracle.mu_of(sigma_r)) + 20
    with mp.workdps(dps):
        mu = oracle.mu_of(sigma_r)
        c = oracle.cheb_c(N, mu, dps)
        nodes = [mp.mpf(mu) * mp.cos(mp.pi * (2 * k - 1) / (2 * (N + 1))) for k in range(1, N + 2)]
        V = mp.matrix([[x ** n for n in range(N + 1)] for x in nodes])
        rhs = mp.matrix([mp.exp(x) for x in nodes])
        sol = mp.lu_solve(V, rhs)
        for n in range(N + 1):
            assert abs(c[n] - sol[n]) <= mp.mpf(10) ** -20 * max(abs(sol[n]), mp.mpf(10) ** -60)


@pytest.mark.parametrize("N,sigma_r", [(n, s) for n, s in STATED + TWINS + PAPER if n % 2 == 0])
def test_c0_is_one_for_even_N(N, sigma_r):
    """Even N: 0 is a node (xi_{N/2+1} = 0), so p(0) = c_0 = e^0 = 1 exactly."""
    c = oracle.cheb_c_float(N, sigma_r)
    assert c[0] == 1.0


def test_c_tends_to_taylor_as_mu_to_zero():
    for N in [3, 8, 12]:
        # c_n n! = 1 + O(mu) (c_N is the divided difference e^zeta / N!, zeta in [-mu, mu])
        c = oracle.cheb_c(N, mp.mpf("1e-12"))
        for n in range(N + 1):
            assert float(c[n]) * math.factorial(n) == pytest.approx(1.0, rel=1e-11)


def test_c_precision_is_converged():
    """Raising the working precision by 40 digits does not change the binary64 c_n."""
    for N, sigma_r in STATED + TWINS:
        mu = oracle.mu_of(sigma_r)
        dps = oracle.required_dps(N, mu)
        c1 = [float(v) for v in oracle.cheb_c(N, mu, dps)]
        c2 = [float(v) for v in oracle.cheb_c(N, mu, dps + 40)]
        assert c1 == c2


def test_taylor_coeffs():
    c = oracle.taylor_c(10)
    assert list(oracle.taylor_c(3)) == [1.0, 1.0, 0.5, 1.0 / 6.0]
    assert abs(math.e - c.sum()) == pytest.approx(math.e - sum(1 / math.factorial(n) for n in range(11)))


def _linf(coeffs, mu, dps=40, npts=801):
    with mp.workdps(dps):
        err = mp.mpf(0)
        for i in range(npts):
            x = mp.mpf(mu) * (-1 + mp.mpf(2 * i) / (npts - 1))
            err = max(err, abs(mp.exp(x) - mp.fsum(coeffs[n] * x ** n for n in range(len(coeffs)))))
        return err


def test_fig1_chebyshev_beats_taylor_and_error_bounds():
    """Fig. 1: on [-1,1] Chebyshev l_inf < Taylor l_inf for N = 2..20.

    Also pinned: Taylor error at N=10 is e - sum_{n<=10} 1/n! (attained at x=1),
    the Chebyshev-node interpolation bound mu^{N+1} e^mu / (2^N (N+1)!), and the
    aliasing bound 4 sum_{l>N} I_l(mu)."""
    lo, hi = GOLD["fig1"]["N_range"]
    for N in range(lo, hi + 1, 2):
        c = oracle.cheb_c(N, 1, 60)
        t = [mp.mpf(1) / mp.factorial(n) for n in range(N + 1)]
        ec, et = _linf(c, 1, npts=401), _linf(t, 1, npts=401)
        assert ec < et, N
        bound = mp.mpf(1) ** (N + 1) * mp.e / (2 ** N * mp.factorial(N + 1))
        assert ec <= bound
        with mp.workdps(40):
            alias = 4 * mp.nsum(lambda l: mp.besseli(l, 1), [N + 1, mp.inf])
        assert ec <= alias
        if N == 10:
            assert float(et) == pytest.approx(math.e - sum(1 / math.factorial(n) for n in range(11)), rel=1e-12)


@pytest.mark.parametrize("N,sigma_r", TWINS)
def test_kernel_error_at_twins_is_small(N, sigma_r):
    """DESIGN.md R1: at the parity twins the degree-N interpolant of exp on [-mu, mu]
    is accurate (relative sup error <= 1e-3 e^mu... measured on the centred kernel)."""
    mu = oracle.mu_of(sigma_r)
    c = oracle.cheb_c(N, mu)
    err = _linf(c, mu, npts=201)
    bound = mu ** (N + 1) * mp.exp(mu) / (2 ** N * mp.factorial(N + 1))
    assert err <= bound
    # Gauss-polynomial kernel sup error sup_{tau,t} e^{-(tau^2+t^2)/2sr^2} |p - exp| <= 1e-3
    with mp.workdps(30):
        worst = mp.mpf(0)
        grid = [mp.mpf(-127.5) + i * mp.mpf(255) / 60 for i in range(61)]
        for tau in grid:
            for tt in grid:
                x = tau * tt / mp.mpf(sigma_r) ** 2
                p = mp.fsum(c[n] * x ** n for n in range(N + 1))
                worst = max(worst, abs(mp.exp(-(tau ** 2 + tt ** 2) / (2 * mp.mpf(sigma_r) ** 2)) * (p - mp.exp(x))))
        assert worst < 1.1e-3
