// gc_operator.cpp — host-side constants of the O(1) exact-window operator (gc_o1.cu).
//
// Eq. (7) filters with the truncated, sampled Gaussian k_m = exp(-m^2/2 sigma_s^2)
// / Z on |m| <= W = ceil(3 sigma_s) (R3, R4, R6).  The O(1) kernels evaluate
// instead  k~_m = sum_{q<K} alpha_q cos(w_q m),  w_q = pi q / Lh,  on exactly the same window,
// so only the coefficients differ.  alpha minimises sum_{|m|<=W} (k~_m - k_m)^2 (normal
// equations in long double); Lh is searched on a grid for the smallest max |k~_m - k_m|.
// With K = 6 the max error is ~1e-6 of the peak tap for every W in 6..4096.
#include <cmath>
#include <map>
#include <mutex>
#include <vector>

#include "gc_internal.h"
#include "gc_lru.h"

namespace gc {
namespace {

// Least-squares alpha for half-period Lh; returns the max abs error of the fit.
double fit_at(const std::vector<double>& k, int W, int K, double Lh, double* alpha) {
  long double A[kO1K][kO1K] = {}, rhs[kO1K] = {};
  std::vector<long double> c(K);
  for (int m = 0; m <= W; m++) {
    const long double w = m == 0 ? 1.0L : 2.0L;           // m and -m both in the window
    for (int q = 0; q < K; q++) c[q] = std::cos((long double)M_PI * q * m / Lh);
    for (int q = 0; q < K; q++) {
      rhs[q] += w * c[q] * k[m];
      for (int r = 0; r < K; r++) A[q][r] += w * c[q] * c[r];
    }
  }
  // Cholesky solve (A is SPD for K <= W+1 and distinct frequencies)
  long double Lc[kO1K][kO1K] = {};
  for (int i = 0; i < K; i++) {
    for (int j = 0; j <= i; j++) {
      long double s = A[i][j];
      for (int t = 0; t < j; t++) s -= Lc[i][t] * Lc[j][t];
      if (i == j) {
        if (!(s > 0)) return INFINITY;
        Lc[i][i] = std::sqrt(s);
      } else {
        Lc[i][j] = s / Lc[j][j];
      }
    }
  }
  long double z[kO1K], x[kO1K];
  for (int i = 0; i < K; i++) {
    long double s = rhs[i];
    for (int t = 0; t < i; t++) s -= Lc[i][t] * z[t];
    z[i] = s / Lc[i][i];
  }
  for (int i = K - 1; i >= 0; i--) {
    long double s = z[i];
    for (int t = i + 1; t < K; t++) s -= Lc[t][i] * x[t];
    x[i] = s / Lc[i][i];
  }
  double err = 0;
  for (int m = 0; m <= W; m++) {
    long double v = 0;
    for (int q = 0; q < K; q++) v += x[q] * std::cos((long double)M_PI * q * m / Lh);
    err = std::max(err, (double)std::fabs(v - k[m]));
  }
  for (int q = 0; q < kO1K; q++) alpha[q] = q < K ? (double)x[q] : 0.0;
  return err;
}

O1Fit compute_fit(float sigma_s) {
  O1Fit f{};
  const int W = (int)std::ceil(3.0 * (double)sigma_s);
  f.R = W;
  std::vector<double> k(W + 1);
  double Z = 0;
  const double ss = (double)sigma_s;
  for (int m = -W; m <= W; m++) Z += std::exp(-(double)m * m / (2.0 * ss * ss));
  for (int m = 0; m <= W; m++) k[m] = std::exp(-(double)m * m / (2.0 * ss * ss)) / Z;
  const int K = std::min(kO1K, W + 1);
  double best = INFINITY, bestL = W + 1.0, alpha[kO1K];
  const int ngrid = 240;
  for (int it = 0; it <= ngrid; it++) {                       // coarse grid on [W + 0.5, 2.5 W + 1]
    const double Lh = (W + 0.5) + (1.5 * W + 0.5) * it / ngrid;
    const double e = fit_at(k, W, K, Lh, alpha);
    if (e < best) { best = e; bestL = Lh; }
  }
  double h = (1.5 * W + 0.5) / ngrid;                          // local refinement
  for (int r = 0; r < 30; r++) {
    h *= 0.5;
    for (double Lh : {bestL - h, bestL + h}) {
      if (Lh <= W) continue;
      const double e = fit_at(k, W, K, Lh, alpha);
      if (e < best) { best = e; bestL = Lh; }
    }
  }
  f.Lh = bestL;
  f.fit_err = fit_at(k, W, K, bestL, f.alpha);
  for (int q = 0; q < kO1K; q++) f.omega[q] = M_PI * q / bestL;
  return f;
}

}  // namespace

O1Fit o1_fit_cached(float sigma_s) {
  static LruMemo<float, O1Fit> cache;       // bounded; computed outside the lock
  return cache.get(sigma_s, [&]() { return compute_fit(sigma_s); });
}

}  // namespace gc
