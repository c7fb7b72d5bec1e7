// mpfloat.h — a small binary multiprecision float for the host coefficient library.
//
// Value = sign * M * 2^e with M an L-limb (32-bit limbs, little endian) integer whose
// top bit is set (normalised) unless the number is zero.  All numbers in one
// computation share the limb count L.  Rounding: truncation after a 2-limb guard in
// add/mul, which the callers absorb with extra guard limbs (see gc_coeffs.cpp).
//
// Only what eqs. (16) and (19) of the paper need: + - * / (small int and general),
// exp, cos, pi, conversion from binary64 / __int128 and correctly-rounded conversion
// back to binary64.  Independent of the oracle (which uses mpmath).
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

namespace gcmp {

class MPF {
 public:
  int sign = 0;                 // 0: zero, +1, -1
  int64_t e = 0;                // exponent of the least significant mantissa bit
  std::vector<uint32_t> m;      // L limbs

  explicit MPF(int L = 4) : m(L, 0u) {}
  int L() const { return (int)m.size(); }
  bool is_zero() const { return sign == 0; }
  // exponent of the value's top bit + 1 (value in [2^(top-1), 2^top))
  int64_t top() const { return e + 32 * (int64_t)m.size(); }
};

// ---------------------------------------------------------------- magnitude helpers

// Normalise an arbitrary-length magnitude `big` (value = big * 2^e) into an L-limb MPF.
inline MPF normalise(std::vector<uint32_t>& big, int64_t e, int sign, int L) {
  MPF r(L);
  int n = (int)big.size();
  int top = n - 1;
  while (top >= 0 && big[top] == 0) top--;
  if (top < 0) { r.sign = 0; r.e = 0; return r; }
  int lz = __builtin_clz(big[top]);
  // total significant bits
  int64_t nbits = 32LL * (top + 1) - lz;
  int64_t shift = nbits - 32LL * L;  // >0: drop low bits; <0: shift left
  // produce r.m = big >> shift (or << -shift)
  if (shift >= 0) {
    int64_t ws = shift / 32; int bs = (int)(shift % 32);
    for (int i = 0; i < L; i++) {
      int64_t s = i + ws;
      uint64_t lo = (s < n) ? big[s] : 0;
      uint64_t hi = (s + 1 < n) ? big[s + 1] : 0;
      uint64_t v = (lo | (hi << 32)) >> bs;
      r.m[i] = (uint32_t)v;
    }
  } else {
    int64_t ls = -shift; int64_t ws = ls / 32; int bs = (int)(ls % 32);
    for (int i = L - 1; i >= 0; i--) {
      int64_t s = i - ws;
      uint64_t hi = (s >= 0 && s < n) ? big[s] : 0;
      uint64_t lo = (s - 1 >= 0 && s - 1 < n) ? big[s - 1] : 0;
      uint64_t v = ((hi << 32) | lo) << bs;
      r.m[i] = (uint32_t)(v >> 32);
    }
  }
  r.e = e + shift;
  r.sign = sign;
  return r;
}

inline int cmp_mag_aligned(const std::vector<uint32_t>& a, const std::vector<uint32_t>& b) {
  for (int i = (int)a.size() - 1; i >= 0; i--) {
    if (a[i] != b[i]) return a[i] > b[i] ? 1 : -1;
  }
  return 0;
}

// ---------------------------------------------------------------- arithmetic

inline MPF add(const MPF& a, const MPF& b) {
  const int L = a.L();
  if (a.is_zero()) return b;
  if (b.is_zero()) return a;
  // If one operand is far below the other's precision, it only affects rounding.
  const int64_t guard_bits = 32LL * (L + 2);
  if (a.top() - b.top() > guard_bits) return a;
  if (b.top() - a.top() > guard_bits) return b;
  int64_t emin = std::max(std::min(a.e, b.e), std::max(a.top(), b.top()) - guard_bits);
  int64_t emax_top = std::max(a.top(), b.top());
  int n = (int)((emax_top - emin) / 32 + 2);
  std::vector<uint32_t> A(n, 0u), B(n, 0u);
  auto place = [&](const MPF& x, std::vector<uint32_t>& X) {
    int64_t sh = x.e - emin;  // may be negative (bits below emin are dropped)
    for (int i = 0; i < L; i++) {
      int64_t bitpos = 32LL * i + sh;
      if (bitpos + 32 <= 0) continue;
      uint64_t v = x.m[i];
      if (bitpos < 0) { v >>= -bitpos; bitpos = 0; }
      int64_t w = bitpos / 32; int bs = (int)(bitpos % 32);
      uint64_t s = v << bs;
      if (w < n) X[w] |= (uint32_t)s;
      if (w + 1 < n) X[w + 1] |= (uint32_t)(s >> 32);
    }
  };
  place(a, A);
  place(b, B);
  std::vector<uint32_t> R(n, 0u);
  int rs;
  if (a.sign == b.sign) {
    uint64_t c = 0;
    for (int i = 0; i < n; i++) { uint64_t s = (uint64_t)A[i] + B[i] + c; R[i] = (uint32_t)s; c = s >> 32; }
    rs = a.sign;
  } else {
    int c = cmp_mag_aligned(A, B);
    if (c == 0) { MPF z(L); return z; }
    const std::vector<uint32_t>& X = c > 0 ? A : B;
    const std::vector<uint32_t>& Y = c > 0 ? B : A;
    int64_t br = 0;
    for (int i = 0; i < n; i++) {
      int64_t s = (int64_t)X[i] - Y[i] - br;
      br = s < 0; if (s < 0) s += (1LL << 32);
      R[i] = (uint32_t)s;
    }
    rs = c > 0 ? a.sign : b.sign;
  }
  return normalise(R, emin, rs, L);
}

inline MPF neg(MPF a) { a.sign = -a.sign; return a; }
inline MPF sub(const MPF& a, const MPF& b) { return add(a, neg(b)); }

inline MPF mul(const MPF& a, const MPF& b) {
  const int L = a.L();
  if (a.is_zero() || b.is_zero()) { MPF z(L); return z; }
  std::vector<uint32_t> P(2 * L, 0u);
  for (int i = 0; i < L; i++) {
    uint64_t c = 0; uint64_t ai = a.m[i];
    for (int j = 0; j < L; j++) {
      uint64_t t = ai * b.m[j] + P[i + j] + c;
      P[i + j] = (uint32_t)t; c = t >> 32;
    }
    P[i + L] = (uint32_t)c;
  }
  return normalise(P, a.e + b.e, a.sign * b.sign, L);
}

inline MPF from_u64(uint64_t v, int L) {
  std::vector<uint32_t> t = {(uint32_t)v, (uint32_t)(v >> 32)};
  return normalise(t, 0, v ? 1 : 0, L);
}

inline MPF from_i128(__int128 v, int L) {
  int s = v > 0 ? 1 : (v < 0 ? -1 : 0);
  unsigned __int128 u = v < 0 ? (unsigned __int128)(-v) : (unsigned __int128)v;
  std::vector<uint32_t> t(4);
  for (int i = 0; i < 4; i++) t[i] = (uint32_t)(u >> (32 * i));
  return normalise(t, 0, s, L);
}

inline MPF from_double(double d, int L) {
  if (d == 0.0) { MPF z(L); return z; }
  int k; double f = std::frexp(std::fabs(d), &k);  // |d| = f * 2^k, f in [0.5, 1)
  uint64_t mi = (uint64_t)std::ldexp(f, 53);        // exact
  MPF r = from_u64(mi, L);
  r.e += k - 53;
  r.sign = d < 0 ? -1 : 1;
  return r;
}

// Correctly rounded (to nearest, ties to even) conversion to binary64 (normal range).
inline double to_double(const MPF& a) {
  if (a.is_zero()) return 0.0;
  const int L = a.L();
  uint64_t t = ((uint64_t)a.m[L - 1] << 32) | (L >= 2 ? a.m[L - 2] : 0u);
  bool sticky = false;
  for (int i = 0; i < L - 2; i++) if (a.m[i]) { sticky = true; break; }
  uint64_t keep = t >> 11, rem = t & 0x7FF;
  if (rem > 0x400 || (rem == 0x400 && (sticky || (keep & 1)))) keep++;
  int64_t ex = a.e + 32LL * L - 64 + 11;
  double v = std::ldexp((double)keep, (int)ex);
  return a.sign < 0 ? -v : v;
}

inline MPF div_small(const MPF& a, uint32_t d) {
  const int L = a.L();
  if (a.is_zero()) return a;
  // divide (a.m << 64) by d to keep full precision
  std::vector<uint32_t> N(L + 2, 0u), Q(L + 2, 0u);
  for (int i = 0; i < L; i++) N[i + 2] = a.m[i];
  uint64_t r = 0;
  for (int i = L + 1; i >= 0; i--) {
    uint64_t cur = (r << 32) | N[i];
    Q[i] = (uint32_t)(cur / d); r = cur % d;
  }
  return normalise(Q, a.e - 64, a.sign, L);
}

inline MPF mul_small(const MPF& a, uint32_t k) { return mul(a, from_u64(k, a.L())); }

inline MPF ldexp(MPF a, int64_t k) { if (!a.is_zero()) a.e += k; return a; }

// 1/b by Newton's iteration x <- x (2 - b x), started from the binary64 reciprocal.
inline MPF recip(const MPF& b) {
  const int L = b.L();
  // scale b to [0.5, 1): b = bs * 2^sh
  int64_t sh = b.top();
  MPF bs = ldexp(b, -sh);
  double approx = 1.0 / to_double(bs);
  MPF x = from_double(approx, L);
  MPF two = from_u64(2, L);
  for (int it = 0; it < 64; it++) {
    MPF nx = mul(x, sub(two, mul(bs, x)));
    MPF diff = sub(nx, x);
    x = nx;
    if (diff.is_zero() || diff.top() < x.top() - 32LL * L + 8) break;
  }
  return ldexp(x, -sh);
}

inline MPF div(const MPF& a, const MPF& b) { return mul(a, recip(b)); }

inline bool negligible(const MPF& term, const MPF& sum) {
  return term.is_zero() || (!sum.is_zero() && term.top() < sum.top() - 32LL * sum.L() - 8);
}

// exp(x): halve the argument s times to |y| < 2^-12, Taylor series, square s times.
inline MPF exp(const MPF& x) {
  const int L = x.L();
  MPF one = from_u64(1, L);
  if (x.is_zero()) return one;
  int64_t s = std::max<int64_t>(0, x.top() + 12);
  MPF y = ldexp(x, -s);
  MPF sum = one, term = one;
  for (uint32_t n = 1; n < 100000; n++) {
    term = div_small(mul(term, y), n);
    sum = add(sum, term);
    if (negligible(term, sum)) break;
  }
  for (int64_t i = 0; i < s; i++) sum = mul(sum, sum);
  return sum;
}

// cos(t), |t| <= 4, by its Taylor series.
inline MPF cos(const MPF& t) {
  const int L = t.L();
  MPF one = from_u64(1, L);
  MPF t2 = mul(t, t);
  MPF sum = one, term = one;
  for (uint32_t n = 1; n < 100000; n++) {
    term = neg(div_small(div_small(mul(term, t2), 2 * n - 1), 2 * n));
    sum = add(sum, term);
    if (negligible(term, sum)) break;
  }
  return sum;
}

// pi by Machin's formula pi = 16 atan(1/5) - 4 atan(1/239).
inline MPF atan_inv(uint32_t x, int L) {
  MPF p = div_small(from_u64(1, L), x);  // x^-(2k+1)
  MPF sum = p;
  const uint32_t x2 = x * x;
  for (uint32_t k = 1; k < 1000000; k++) {
    p = div_small(p, x2);
    MPF t = div_small(p, 2 * k + 1);
    sum = (k & 1) ? sub(sum, t) : add(sum, t);
    if (negligible(t, sum)) break;
  }
  return sum;
}

inline MPF pi(int L) {
  return sub(mul_small(atan_inv(5, L), 16), mul_small(atan_inv(239, L), 4));
}

inline MPF abs(MPF a) { if (a.sign < 0) a.sign = 1; return a; }
inline bool less_mag(const MPF& a, const MPF& b) {  // |a| < |b|
  if (a.is_zero()) return !b.is_zero();
  if (b.is_zero()) return false;
  if (a.top() != b.top()) return a.top() < b.top();
  for (int i = a.L() - 1; i >= 0; i--) if (a.m[i] != b.m[i]) return a.m[i] < b.m[i];
  return false;
}

}  // namespace gcmp
