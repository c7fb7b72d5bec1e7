// gc_coeffs.cpp — host coefficient library.
//
// c_n of eq. (19) for the degree-N Chebyshev interpolant of exp on
// [-mu, mu] (eq. 16 rescaled), mu = (U-L)^2 / (4 sigma_r^2),
// evaluated in gcmp::MPF multiprecision (mpfloat.h) and rounded once to binary64.
//
// Why extended precision (R2): eq. (19) cancels terms of size ~e^mu 2^N down to
// c_n mu^n, which can be O(1); eq. (16) cancels O(1) samples down to d_l ~ (mu/2)^l / l!
// when mu is small.  The working precision covers both plus 128 guard bits.
//
// Also produces the fp32 kernel constants (gc_internal.h GcCoefs):
//   chat_n = c_n mu^n / max_m |c_m mu^m|      (= sum_l d_l a_{l,n}, normalised)
// which multiply the scaled planes  G'_n = (g/t_h)^n,  F'_n = exp(-g^2/2sr^2) (g/t_h)^n,
// t_h = (U-L)/2, because c_n G_n Fbar_n = c_n mu^n G'_n Fbar'_n  (t_h/sigma_r = sqrt(mu)).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include "gc_internal.h"
#include "gc_lru.h"
#include "mpfloat.h"

using gcmp::MPF;

namespace {

int limbs_for(int N, double mu) {
  double small = mu > 0 ? N * std::max(0.0, std::log10(1.0 / mu)) : 0.0;
  double digits = 40.0 + mu / std::log(10.0) + N * std::log10(2.0) + small;
  double bits = digits * 3.3219280948873623 + 128.0;
  return (int)std::ceil(bits / 32.0) + 2;
}

// T_l coefficients a_{l,n} (eq. 13) from the recursion induced by eq. (12):
// a_{l+1,n} = 2 a_{l,n-1} - a_{l-1,n}.  |a_{64,n}| < 2^90, so __int128 is exact.
std::vector<std::vector<__int128>> monomial_table(int N) {
  std::vector<std::vector<__int128>> a(N + 1);
  a[0] = {1};
  if (N >= 1) a[1] = {0, 1};
  for (int l = 1; l < N; l++) {
    a[l + 1].assign(l + 2, 0);
    for (int n = 0; n <= l + 1; n++) {
      __int128 up = (n >= 1 && n - 1 <= l) ? 2 * a[l][n - 1] : 0;
      __int128 down = (n <= l - 1) ? a[l - 1][n] : 0;
      a[l + 1][n] = up - down;
    }
  }
  return a;
}

struct CoefResult {
  std::vector<double> c;       // c_n, binary64
  std::vector<double> cmu;     // c_n mu^n / max |c_m mu^m|, binary64
  double mu;
};

CoefResult compute(int N, double sigma_r, double L, double U) {
  const double mu_d = (U - L) * (U - L) / (4.0 * sigma_r * sigma_r);
  const int LB = limbs_for(N, mu_d);
  // mu exactly from the binary64 inputs: (U-L)^2 / (4 sigma_r^2)
  MPF uml = gcmp::sub(gcmp::from_double(U, LB), gcmp::from_double(L, LB));
  MPF sr = gcmp::from_double(sigma_r, LB);
  MPF mu = gcmp::div(gcmp::mul(uml, uml), gcmp::ldexp(gcmp::mul(sr, sr), 2));

  // cos(pi q / (2(N+1))), q = 0..2(N+1): every T_l(xi_k) = cos(l theta_k) with
  // theta_k = pi (2k-1) / (2(N+1)) reduces to one of these (cos is even, 2pi-periodic).
  const int M = N + 1;
  MPF pi = gcmp::pi(LB);
  std::vector<MPF> C(2 * M + 1, MPF(LB));
  for (int q = 0; q <= 2 * M; q++) {
    MPF ang = gcmp::div_small(gcmp::mul_small(pi, (uint32_t)q), (uint32_t)(2 * M));
    C[q] = gcmp::cos(ang);
  }
  // h_k = exp(mu xi_k), xi_k = cos(theta_k) = C[2k-1], k = 1..N+1
  std::vector<MPF> h(M + 1, MPF(LB));
  for (int k = 1; k <= M; k++) h[k] = gcmp::exp(gcmp::mul(mu, C[2 * k - 1]));
  // d_l
  std::vector<MPF> d(N + 1, MPF(LB));
  for (int l = 0; l <= N; l++) {
    MPF s(LB);
    for (int k = 1; k <= M; k++) {
      long q = ((long)l * (2 * k - 1)) % (4 * M);
      if (q > 2 * M) q = 4 * M - q;
      s = gcmp::add(s, gcmp::mul(h[k], C[q]));
    }
    d[l] = (l == 0) ? gcmp::div_small(s, (uint32_t)M) : gcmp::div_small(gcmp::ldexp(s, 1), (uint32_t)M);
  }
  // c_n mu^n = sum_{l=n}^{N} d_l a_{l,n}   (eq. 19 before the division by mu^n)
  auto a = monomial_table(N);
  std::vector<MPF> cm(N + 1, MPF(LB));
  for (int n = 0; n <= N; n++) {
    MPF s(LB);
    for (int l = n; l <= N; l++) {
      if (a[l][n] == 0) continue;
      s = gcmp::add(s, gcmp::mul(d[l], gcmp::from_i128(a[l][n], LB)));
    }
    cm[n] = s;
  }
  CoefResult r;
  r.mu = gcmp::to_double(mu);
  r.c.resize(N + 1);
  r.cmu.resize(N + 1);
  MPF rmu = gcmp::recip(mu);
  MPF pw = gcmp::from_u64(1, LB);
  MPF mx(LB);
  for (int n = 0; n <= N; n++) {
    r.c[n] = gcmp::to_double(gcmp::mul(cm[n], pw));   // c_n = (1/mu)^n (...)
    pw = gcmp::mul(pw, rmu);
    if (gcmp::less_mag(mx, cm[n])) mx = gcmp::abs(cm[n]);
  }
  MPF rmx = gcmp::recip(mx);
  for (int n = 0; n <= N; n++) r.cmu[n] = gcmp::to_double(gcmp::mul(cm[n], rmx));
  return r;
}

gc::LruMemo<std::tuple<int, uint64_t, uint64_t, uint64_t>, CoefResult> g_cache;   // bounded

uint64_t bits_of(double x) { uint64_t b; std::memcpy(&b, &x, 8); return b; }

}  // namespace

namespace gc {

gc_status coeffs_cached(int N, double sigma_r, double L, double U, std::vector<double>* c,
                        std::vector<double>* cmu, double* mu) {
  if (N < 0 || !(sigma_r > 0) || !(U > L) || !std::isfinite(sigma_r) || !std::isfinite(L) || !std::isfinite(U))
    return GC_EINVAL;
  if (N > GC_N_MAX) return GC_ERANGE;
  const double mu_d = (U - L) * (U - L) / (4.0 * sigma_r * sigma_r);
  if (!(mu_d <= GC_MU_MAX)) return GC_ERANGE;
  if (!(mu_d > 1e-30)) return GC_ERANGE;
  auto key = std::make_tuple(N, bits_of(sigma_r), bits_of(L), bits_of(U));
  const CoefResult r = g_cache.get(key, [&]() { return compute(N, sigma_r, L, U); });
  if (c) *c = r.c;
  if (cmu) *cmu = r.cmu;
  if (mu) *mu = r.mu;
  return GC_OK;
}

}  // namespace gc

extern "C" gc_status gc_coeffs(int N, double sigma_r, double L, double U, double* c_out, double* mu_out) {
  if (!c_out) return GC_EINVAL;
  std::vector<double> c;
  double mu = 0;
  gc_status st = gc::coeffs_cached(N, sigma_r, L, U, &c, nullptr, &mu);
  if (st != GC_OK) return st;
  std::memcpy(c_out, c.data(), sizeof(double) * (N + 1));
  if (mu_out) *mu_out = mu;
  return GC_OK;
}
