// gc_operator.cpp — host-side constants of the O(1) exact-window operator (gc_o1.cu).
//
// Eq. (7) filters with the truncated, sampled Gaussian k_m = exp(-m^2/2 sigma_s^2)
// / Z on |m| <= W = ceil(3 sigma_s) (R3, R4, R6).  The O(1) kernels evaluate
// instead  k~_m = sum_{q<K} alpha_q cos(w_q m)  on exactly the same window (w_0 = 0: the box
// term), so only the coefficients differ.
//
// Round 2: the frequencies w_1..w_{K-1} are free parameters, not a harmonic series pi q / Lh.
// For given frequencies alpha is the weighted least-squares solution (normal equations in long
// double, "variable projection"); the frequencies are refined by Gauss-Newton steps on the
// residual, inside an iteratively reweighted loop (Lawson) that drives the fit from least squares
// towards the minimax (max-error) solution.  With K = 5 (box + 4 resonators) the max error is
// ~5e-8 of the peak tap for every W (the harmonic K = 6 fit of round 1: ~7e-7), so the kernels
// run one resonator fewer per plane-sample and pass.
#include <algorithm>
#include <cmath>
#include <map>
#include <mutex>
#include <vector>

#include "gc_internal.h"
#include "gc_lru.h"

namespace gc {
namespace {

typedef long double LD;

// Weighted least-squares alpha for frequencies om[0..K-1] on samples m = 0..W with weights wt
// (the symmetric count times the Lawson weights); residual r_m = sum alpha_q cos(om_q m) - k_m.
// Returns false if the normal equations are singular.
bool ls_alpha(const std::vector<LD>& k, const std::vector<LD>& wt, int W, int K, const LD* om, LD* alpha,
              std::vector<LD>* r) {
  LD A[kO1K][kO1K] = {}, rhs[kO1K] = {};
  LD c[kO1K];
  for (int m = 0; m <= W; m++) {
    for (int q = 0; q < K; q++) c[q] = std::cos(om[q] * m);
    for (int q = 0; q < K; q++) {
      rhs[q] += wt[m] * c[q] * k[m];
      for (int t = 0; t < K; t++) A[q][t] += wt[m] * c[q] * c[t];
    }
  }
  LD Lc[kO1K][kO1K] = {};
  for (int i = 0; i < K; i++) {
    for (int j = 0; j <= i; j++) {
      LD s = A[i][j];
      for (int t = 0; t < j; t++) s -= Lc[i][t] * Lc[j][t];
      if (i == j) {
        if (!(s > 1e-300L)) return false;
        Lc[i][i] = std::sqrt(s);
      } else {
        Lc[i][j] = s / Lc[j][j];
      }
    }
  }
  LD z[kO1K];
  for (int i = 0; i < K; i++) {
    LD s = rhs[i];
    for (int t = 0; t < i; t++) s -= Lc[i][t] * z[t];
    z[i] = s / Lc[i][i];
  }
  for (int i = K - 1; i >= 0; i--) {
    LD s = z[i];
    for (int t = i + 1; t < K; t++) s -= Lc[t][i] * alpha[t];
    alpha[i] = s / Lc[i][i];
  }
  if (r) {
    r->resize(W + 1);
    for (int m = 0; m <= W; m++) {
      LD v = 0;
      for (int q = 0; q < K; q++) v += alpha[q] * std::cos(om[q] * m);
      (*r)[m] = v - k[m];
    }
  }
  return true;
}

LD max_abs(const std::vector<LD>& r) {
  LD e = 0;
  for (LD v : r) e = std::max(e, std::fabs(v));
  return e;
}

// Solve the small dense system J^T W J d = -J^T W r (Gauss-Newton normal equations) for the
// free frequencies; returns false if singular.
bool gn_step(const std::vector<std::vector<LD>>& J, const std::vector<LD>& r, const std::vector<LD>& wt, int n,
             LD* d) {
  const int P = (int)J.size();
  LD M[kO1K][kO1K + 1] = {};
  for (int m = 0; m < n; m++)
    for (int a = 0; a < P; a++) {
      M[a][P] -= wt[m] * J[a][m] * r[m];
      for (int b = 0; b < P; b++) M[a][b] += wt[m] * J[a][m] * J[b][m];
    }
  for (int a = 0; a < P; a++) M[a][a] *= 1.0L + 1e-9L;      // (tiny Levenberg damping)
  for (int c = 0; c < P; c++) {                             // Gaussian elimination, partial pivoting
    int piv = c;
    for (int a = c + 1; a < P; a++)
      if (std::fabs(M[a][c]) > std::fabs(M[piv][c])) piv = a;
    if (!(std::fabs(M[piv][c]) > 1e-300L)) return false;
    if (piv != c)
      for (int b = 0; b <= P; b++) std::swap(M[c][b], M[piv][b]);
    for (int a = c + 1; a < P; a++) {
      const LD f = M[a][c] / M[c][c];
      for (int b = c; b <= P; b++) M[a][b] -= f * M[c][b];
    }
  }
  for (int a = P - 1; a >= 0; a--) {
    LD s = M[a][P];
    for (int b = a + 1; b < P; b++) s -= M[a][b] * d[b];
    d[a] = s / M[a][a];
  }
  return true;
}

LD wss(const std::vector<LD>& wt, const std::vector<LD>& r) {
  LD s = 0;
  for (size_t m = 0; m < r.size(); m++) s += wt[m] * r[m] * r[m];
  return s;
}

O1Fit compute_fit(float sigma_s) {
  O1Fit f{};
  const int W = (int)std::ceil(3.0 * (double)sigma_s);
  f.R = W;
  std::vector<LD> k(W + 1), sym(W + 1), wt(W + 1), r;
  LD Z = 0;
  const LD ss = (LD)sigma_s;
  for (int m = -W; m <= W; m++) Z += std::exp(-(LD)m * m / (2.0L * ss * ss));
  for (int m = 0; m <= W; m++) {
    k[m] = std::exp(-(LD)m * m / (2.0L * ss * ss)) / Z;
    sym[m] = m == 0 ? 1.0L : 2.0L;                          // m and -m both in the window
  }
  const int K = std::min(kO1K, W + 1);
  LD om[kO1K] = {}, alpha[kO1K] = {};
  // the minimax frequencies scale as w_q = c_q pi / W for large W; c_q from this optimisation at
  // W = 4095 (the W = 1200 optimum agrees to 5e-6).  They are the starting point for small W and
  // used as they are above kO1FitFree (the optimisation costs O(W) per iteration; measured max
  // error with the fixed c_q: ~5e-8 of the peak tap, tests/test_abi.py::test_operator_taps)
  constexpr int kO1FitFree = 64;
  const LD c0[4] = {0.867920910L, 1.759659631L, 2.710096021L, 3.799544073L};
  for (int q = 1; q < K; q++) om[q] = std::min<LD>(c0[q - 1] * (LD)M_PI / (LD)std::max(W, 1), (LD)M_PI * q / K);
  if (K <= W && W <= kO1FitFree) {
    // Lawson-reweighted least squares with Gauss-Newton refinement of the frequencies
    std::vector<LD> law(W + 1, 1.0L);
    LD best_err = INFINITY, best_om[kO1K] = {};
    for (int it = 0; it < 40; it++) {
      for (int m = 0; m <= W; m++) wt[m] = sym[m] * law[m];
      for (int gn = 0; gn < 4; gn++) {
        if (!ls_alpha(k, wt, W, K, om, alpha, &r)) break;
        // numerical Jacobian of the residual (alpha re-solved: variable projection)
        std::vector<std::vector<LD>> J(K - 1, std::vector<LD>(W + 1));
        bool ok = true;
        for (int q = 1; q < K && ok; q++) {
          LD om2[kO1K], a2[kO1K];
          std::copy(om, om + K, om2);
          const LD h = 1e-7L * std::max(om[q], (LD)1e-3);
          om2[q] += h;
          std::vector<LD> r2;
          ok = ls_alpha(k, wt, W, K, om2, a2, &r2);
          for (int m = 0; m <= W && ok; m++) J[q - 1][m] = (r2[m] - r[m]) / h;
        }
        LD d[kO1K] = {};
        if (!ok || !gn_step(J, r, wt, W + 1, d)) break;
        const LD cur = wss(wt, r);                          // damped step: accept if not worse
        LD step = 1.0L;
        for (int tries = 0; tries < 20; tries++, step *= 0.5L) {
          LD om2[kO1K], a2[kO1K];
          std::copy(om, om + K, om2);
          bool sane = true;
          for (int q = 1; q < K; q++) {
            om2[q] += step * d[q - 1];
            if (!(om2[q] > 0 && om2[q] < (LD)M_PI)) sane = false;
          }
          std::vector<LD> r2;
          if (!sane || !ls_alpha(k, wt, W, K, om2, a2, &r2)) continue;
          if (wss(wt, r2) <= cur) {
            std::copy(om2, om2 + K, om);
            break;
          }
        }
      }
      if (!ls_alpha(k, sym, W, K, om, alpha, &r)) break;   // plain least squares at these frequencies
      const LD e = max_abs(r);
      if (e < best_err) {
        best_err = e;
        std::copy(om, om + K, best_om);
      }
      // Lawson update towards the minimax fit, on the current weighted residual
      if (!ls_alpha(k, wt, W, K, om, alpha, &r)) break;
      LD mean = 0;
      for (int m = 0; m <= W; m++) mean += (law[m] *= std::fabs(r[m]) + 1e-30L);
      mean /= (W + 1);
      if (!(mean > 0)) break;
      for (int m = 0; m <= W; m++) law[m] /= mean;
    }
    if (best_err < INFINITY) std::copy(best_om, best_om + K, om);
  }
  ls_alpha(k, sym, W, K, om, alpha, &r);      // W + 1 <= K: the samples are interpolated exactly
  f.fit_err = (double)max_abs(r);
  for (int q = 0; q < kO1K; q++) {
    f.alpha[q] = q < K ? (double)alpha[q] : 0.0;
    f.omega[q] = q < K ? (double)om[q] : 0.0;
  }
  f.Lh = 0;
  return f;
}

}  // namespace

O1Fit o1_fit_cached(float sigma_s) {
  static LruMemo<float, O1Fit> cache;       // bounded; computed outside the lock
  return cache.get(sigma_s, [&]() { return compute_fit(sigma_s); });
}

}  // namespace gc
