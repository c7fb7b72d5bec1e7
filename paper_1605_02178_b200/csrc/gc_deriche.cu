// gc_deriche.cu — the Deriche-class recursive "fast mode" (GC_OP_DERICHE)
// for the N+2 spatial filterings of the GCF.
//
// PAPER P:50 and P:112 reach O(1) cost per pixel for eq. (7) "using separability and
// recursion" and cite Deriche's recursive Gaussian [Deriche1993].  That filter is the
// untruncated 4th-order fit
//     h(x) = (a0 cos(w0 x/s) + a1 sin(w0 x/s)) e^{-b0 x/s} + (c0 cos(w1 x/s) + c1 sin(w1 x/s)) e^{-b1 x/s}
// applied as a causal recursion (impulse response h(k), k >= 0) plus an anticausal one
// (h(k), k >= 1), normalised by Z = sum_k h(|k|), on each line padded with K = ceil(10 s)
// whole-sample mirrored samples per side and started from zero state (R15; the
// binary64 oracle is oracle/deriche.py, which runs the same filter as one 4th-order
// direct-form recursion).  It is NOT eq. (7): the GCF moves by ~0.2-0.35 grey levels
// (SURVEY A.5), which is why it is a separate, opt-in operator.
//
// fp32 design: each direction is the sum of two real 2nd-order sections, one per complex-
// conjugate pole pair q_j = exp((-b_j + i w_j)/s) (partial fractions of the 4th-order
// recursion; 1/Z folded into the numerators):
//     causal      v[k] = b0 x[k] + b1 x[k-1] + a1 v[k-1] - a2 v[k-2]
//     anticausal  w[k] = c1 x[k+1] + c2 x[k+2] + a1 w[k+1] - a2 w[k+2],   a1 = 2 Re q, a2 = |q|^2
// The 4th-order direct form loses 3e-4 (s = 16) to 9e-3 (s = 40) relative in fp32; the
// sections stay at 3e-6 / 1.1e-5 (prototype vs the binary64 oracle).
//
// Both passes put one LINE per lane and sweep along it: a line is split into segments; a
// segment's causal sweep starts from zero state K samples before its first output (or at
// the padded edge -K, exactly like the oracle) and its anticausal sweep K samples after its
// last output (or at n-1+K); the zero-state start differs from the oracle's by |q|^K ~ 3e-8.
// The two directions meet at every output, so the causal partial sums of a segment are
// stored (global scratch, coalesced) and added during the anticausal sweep:
//   k_row_dr   lane = image row (32 rows per warp), all NP plane pairs of the row: planes are
//              generated from f on the fly (eq. 6) for both sweeps; causal sums go to the
//              scratch in [B][NP][Wd][rows] order (lane-contiguous); the filtered pairs are
//              staged through shared memory in 8-column chunks and stored as rows of the plane
//              buffer [B][NP][rows][Wd].
//   k_col_dr   lane = image column: causal sweep down the column (plane rows read coalesced),
//              partial sums to the scratch [B][NP][out_rows][Wd]; anticausal sweep up, plus the
//              recombination of eqs. (8)-(10) with the guard of DESIGN.md R8.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <complex>
#include <cstring>

#include "gc_device.cuh"

namespace gc {

constexpr int kDrWarps = 4;          // warps per CTA (independent tasks)
constexpr int kDrChunk = 8;          // row pass: output columns per shared-memory flush

// ------------------------------------------------------------------ host: coefficients

// Deriche (1993) 4th-order fit of exp(-x^2/2): (a0, a1, b0, w0) and (c0, c1, b1, w1).
static const double kDer[2][4] = {{1.68, 3.735, 1.783, 0.6318}, {-0.6803, -0.2598, 1.723, 1.997}};

void deriche_constants(float sigma_s, KParams& k) {
  const double s = (double)sigma_s;
  double Z = 0;
  std::complex<double> r[2], q[2];
  for (int j = 0; j < 2; j++) {
    r[j] = std::complex<double>(kDer[j][0], -kDer[j][1]) * 0.5;
    q[j] = std::exp(std::complex<double>(-kDer[j][2], kDer[j][3]) / s);
    // sum_{k in Z} 2 Re(r q^|k|) = 2 Re(r (1 + q) / (1 - q))
    Z += 2.0 * std::real(r[j] * (1.0 + q[j]) / (1.0 - q[j]));
  }
  for (int j = 0; j < 2; j++) {
    auto g = [&](int n) { return 2.0 * std::real(r[j] * std::pow(q[j], n)); };   // section impulse response
    const double a1 = 2.0 * std::real(q[j]), a2 = std::norm(q[j]);
    k.dr_a1[j] = (float)a1;
    k.dr_a2[j] = (float)a2;
    k.dr_b0[j] = (float)(g(0) / Z);
    k.dr_b1[j] = (float)((g(1) - a1 * g(0)) / Z);
    k.dr_c1[j] = (float)(g(1) / Z);
    k.dr_c2[j] = (float)((g(2) - a1 * g(1)) / Z);
  }
  k.dr_K = (int)std::ceil(10.0 * s);
}

// ------------------------------------------------------------------ device helpers

// One step of the causal sections on a plane pair: returns v0 + v1 and advances the state.
struct DrCausal {
  float2 v1[2], v2[2], xm;
  __device__ __forceinline__ void zero() {
    v1[0] = v1[1] = v2[0] = v2[1] = xm = make_float2(0.f, 0.f);
  }
  __device__ __forceinline__ float2 step(const KParams& p, float2 x) {
    float2 y = make_float2(0.f, 0.f);
#pragma unroll
    for (int j = 0; j < 2; j++) {
      float2 v = f2mul(f2s(p.dr_b0[j]), x);
      v = f2fma(f2s(p.dr_b1[j]), xm, v);
      v = f2fma(f2s(p.dr_a1[j]), v1[j], v);
      v = f2fma(f2s(-p.dr_a2[j]), v2[j], v);
      v2[j] = v1[j];
      v1[j] = v;
      y = f2add(y, v);
    }
    xm = x;
    return y;
  }
};

// One step of the anticausal sections (x = the sample at k; returns w[k], which uses
// x[k+1], x[k+2] only) and advances the state.
struct DrAnti {
  float2 w1[2], w2[2], x1, x2;
  __device__ __forceinline__ void zero() {
    w1[0] = w1[1] = w2[0] = w2[1] = x1 = x2 = make_float2(0.f, 0.f);
  }
  __device__ __forceinline__ float2 step(const KParams& p, float2 x) {
    float2 y = make_float2(0.f, 0.f);
#pragma unroll
    for (int j = 0; j < 2; j++) {
      float2 w = f2mul(f2s(p.dr_c1[j]), x1);
      w = f2fma(f2s(p.dr_c2[j]), x2, w);
      w = f2fma(f2s(p.dr_a1[j]), w1[j], w);
      w = f2fma(f2s(-p.dr_a2[j]), w2[j], w);
      w2[j] = w1[j];
      w1[j] = w;
      y = f2add(y, w);
    }
    x2 = x1;
    x1 = x;
    return y;
  }
};

// Plane pairs (F'_{2q}, F'_{2q+1}), q < NPG, of one input sample (eq. 6 with the scaling of
// DESIGN.md §3): psi_0 = e (1, a'), psi_{q+1} = psi_q a'^2.  raw: pair 0 = (f, 0).
template <int NPG>
__device__ __forceinline__ void dr_planes(const KParams& p, float f, float2 (&psi)[NPG]) {
  float a, e;
  centre(p, f, a, e);
  if (p.raw) {
    psi[0] = make_float2(f, 0.f);
  } else {
    psi[0] = make_float2(e, e * a);
  }
  const float2 a2 = f2s(a * a);
#pragma unroll
  for (int q = 1; q < NPG; q++) psi[q] = f2mul(psi[q - 1], a2);
}

// ------------------------------------------------------------------ row pass

struct DrRowSmem {
  float2 tile[kDrMaxPairs][32][kDrChunk + 1];   // [pair][row][column in chunk] (padded: bank spread)
};

template <int NPG>
__global__ void __launch_bounds__(32 * kDrWarps) k_row_dr(const KParams p) {
  pdl_trigger();
  extern __shared__ __align__(16) float4 smem_dr[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  DrRowSmem& sm = reinterpret_cast<DrRowSmem*>(smem_dr)[warp];
  const int nrb = (p.in_rows + 31) / 32;
  const int ntask = nrb * p.dr_nseg_x * p.B;
  const int task = blockIdx.x * kDrWarps + warp;
  if (task >= ntask) return;
  const int rb = task % nrb;
  const int sx = (task / nrb) % p.dr_nseg_x;
  const int b = task / (nrb * p.dr_nseg_x);
  const int n = p.Wd, K = p.dr_K;
  const int x0 = sx * p.dr_seg_x, x1 = min(x0 + p.dr_seg_x, n);
  const int row = rb * 32 + lane;
  const bool rok = row < p.in_rows;
  const int rowc = rok ? row : p.in_rows - 1;
  const float* src = row_ptr(p, b, p.in_row0 + rowc);
  // causal partial sums: scratch [B][NP][Wd][in_rows] (lane-contiguous)
  float2* const yp = p.scratch + (long long)b * p.NP * n * p.in_rows + rowc;
  const long long yp_pair = (long long)n * p.in_rows;

  // f of this lane's row, 8 consecutive padded positions at a time (the next group's loads are
  // issued before the current group's recursions)
  auto load8 = [&](int c, float (&v)[8]) {
#pragma unroll
    for (int i = 0; i < 8; i++) {
      GC_CHK(p, src + mirror(c + i, n), 4);
      v[i] = __ldg(src + mirror(c + i, n));
    }
  };

  // ---- causal sweep, padded coordinates c in [cs0, x1), cs0 = max(x0 - K, -K)
  DrCausal cs[NPG];
#pragma unroll
  for (int q = 0; q < NPG; q++) cs[q].zero();
  {
    const int cs0 = max(x0 - K, -K);
    float fc[8], fn[8];
    load8(cs0, fn);
#pragma unroll 1
    for (int c8 = cs0; c8 < x1; c8 += 8) {
#pragma unroll
      for (int i = 0; i < 8; i++) fc[i] = fn[i];
      if (c8 + 8 < x1) load8(c8 + 8, fn);
#pragma unroll
      for (int i = 0; i < 8; i++) {
        const int c = c8 + i;
        if (c >= x1) break;
        float2 psi[NPG];
        dr_planes<NPG>(p, fc[i], psi);
#pragma unroll
        for (int q = 0; q < NPG; q++) {
          const float2 y = cs[q].step(p, psi[q]);
          if (c >= x0 && rok) {
            GC_CHK(p, &yp[q * yp_pair + (long long)c * p.in_rows], 8);
            yp[q * yp_pair + (long long)c * p.in_rows] = y;
          }
        }
      }
    }
  }

  // ---- anticausal sweep, c from min(x1 + K, n + K) - 1 down to x0: lead-in, then the outputs
  //      in 8-column chunks (f for the next 8 positions and the causal sums for the next
  //      position prefetched)
  DrAnti as[NPG];
#pragma unroll
  for (int q = 0; q < NPG; q++) as[q].zero();
  const int cstart = min(x1 + K, n + K) - 1;
  {
    float fc[8], fn[8];
    if (cstart >= x1) load8(cstart - 7, fn);
#pragma unroll 1
    for (int c8 = cstart; c8 >= x1; c8 -= 8) {   // positions c8, c8-1, .., c8-7 (>= x1)
#pragma unroll
      for (int i = 0; i < 8; i++) fc[i] = fn[i];
      if (c8 - 8 >= x1) load8(c8 - 15, fn);
#pragma unroll
      for (int i = 7; i >= 0; i--) {
        const int c = c8 - 7 + i;
        if (c < x1) break;
        float2 psi[NPG];
        dr_planes<NPG>(p, fc[i], psi);
#pragma unroll
        for (int q = 0; q < NPG; q++) as[q].step(p, psi[q]);
      }
    }
  }
  float2* const dst = p.planes + b * p.planes_img_stride;
  const long long pstride = (long long)p.in_rows * n;
  const int nchunk = (x1 - x0 + kDrChunk - 1) / kDrChunk;
  float2 ypn[NPG];
#pragma unroll
  for (int q = 0; q < NPG; q++) {
    GC_CHK(p, &yp[q * yp_pair + (long long)(x1 - 1) * p.in_rows], 8);
    ypn[q] = yp[q * yp_pair + (long long)(x1 - 1) * p.in_rows];
  }
#pragma unroll 1
  for (int ch = nchunk - 1; ch >= 0; ch--) {
    const int c0 = x0 + ch * kDrChunk, c1 = min(c0 + kDrChunk, x1);
    float fc[8];
    load8(c0, fc);
#pragma unroll
    for (int i = kDrChunk - 1; i >= 0; i--) {
      const int c = c0 + i;
      if (c >= c1) continue;
      float2 ypc[NPG];
#pragma unroll
      for (int q = 0; q < NPG; q++) ypc[q] = ypn[q];
      if (c > x0) {
#pragma unroll
        for (int q = 0; q < NPG; q++) {
          GC_CHK(p, &yp[q * yp_pair + (long long)(c - 1) * p.in_rows], 8);
          ypn[q] = yp[q * yp_pair + (long long)(c - 1) * p.in_rows];
        }
      }
      float2 psi[NPG];
      dr_planes<NPG>(p, fc[i], psi);
#pragma unroll
      for (int q = 0; q < NPG; q++) sm.tile[q][lane][i] = f2add(as[q].step(p, psi[q]), ypc[q]);
    }
    __syncwarp();
    // rows of the chunk: lane -> (row r = lane / 8 + 4 i, column j = lane % 8)
    const int j = lane % kDrChunk;
#pragma unroll
    for (int q = 0; q < NPG; q++) {
      if (q >= p.NP) break;
#pragma unroll
      for (int i = 0; i < 4; i++) {
        const int r = lane / kDrChunk + 4 * i;
        const int rr = rb * 32 + r;
        // (rows r + 16 .. r + 28 are handled by the second half below)
        if (rr < p.in_rows && c0 + j < c1) {
          GC_CHK(p, &dst[q * pstride + (long long)rr * n + c0 + j], 8);
          dst[q * pstride + (long long)rr * n + c0 + j] = sm.tile[q][r][j];
        }
        const int r2 = r + 16, rr2 = rb * 32 + r2;
        if (rr2 < p.in_rows && c0 + j < c1) {
          GC_CHK(p, &dst[q * pstride + (long long)rr2 * n + c0 + j], 8);
          dst[q * pstride + (long long)rr2 * n + c0 + j] = sm.tile[q][r2][j];
        }
      }
    }
    __syncwarp();
  }
}

// ------------------------------------------------------------------ column pass

template <int NPG>
__global__ void __launch_bounds__(32 * kDrWarps) k_col_dr(const KParams p) {
  pdl_wait();                                      // planes from k_row_dr
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ncb = (p.Wd + 31) / 32;
  const int ntask = ncb * p.dr_nseg_y * p.B;
  const int task = blockIdx.x * kDrWarps + warp;
  if (task >= ntask) return;
  const int cb = task % ncb;
  const int sy = (task / ncb) % p.dr_nseg_y;
  const int b = task / (ncb * p.dr_nseg_y);
  const int x = cb * 32 + lane;
  const bool xok = x < p.Wd;
  const int xc = xok ? x : p.Wd - 1;
  const int H = p.H, K = p.dr_K;
  const int y0 = sy * p.dr_seg_y, y1 = min(y0 + p.dr_seg_y, p.out_rows);   // output rows (window)
  const int g0 = p.out_row0 + y0, g1 = p.out_row0 + y1;                   // global rows
  const long long pstride = (long long)p.in_rows * p.Wd;
  const float2* const pl = p.planes + b * p.planes_img_stride + xc;
  float2* const ys = p.scratch + (long long)b * p.NP * p.out_rows * p.Wd + xc;   // [NP][out_rows][Wd]
  const long long ys_pair = (long long)p.out_rows * p.Wd;
  auto prow = [&](int g) { return (long long)(mirror(g, H) - p.in_row0) * p.Wd; };

  // ---- causal sweep down: global rows g in [max(g0 - K, -K), g1), 2 rows per iteration
  //      (loads of the next row issued before the current row's recursion)
  DrCausal cs[NPG];
#pragma unroll
  for (int q = 0; q < NPG; q++) cs[q].zero();
  {
    const int gs = max(g0 - K, -K);
    float2 nx[NPG];
#pragma unroll
    for (int q = 0; q < NPG; q++) {
      GC_CHK(p, pl + q * pstride + prow(gs), 8);
      nx[q] = __ldg(pl + q * pstride + prow(gs));
    }
#pragma unroll 1
    for (int g = gs; g < g1; g++) {
      float2 cx[NPG];
#pragma unroll
      for (int q = 0; q < NPG; q++) cx[q] = nx[q];
      if (g + 1 < g1) {
        const long long o = prow(g + 1);
#pragma unroll
        for (int q = 0; q < NPG; q++) {
          GC_CHK(p, pl + q * pstride + o, 8);
          nx[q] = __ldg(pl + q * pstride + o);
        }
      }
#pragma unroll
      for (int q = 0; q < NPG; q++) {
        const float2 y = cs[q].step(p, cx[q]);
        if (g >= g0) {
          GC_CHK(p, &ys[q * ys_pair + (long long)(g - p.out_row0) * p.Wd], 8);
          ys[q * ys_pair + (long long)(g - p.out_row0) * p.Wd] = y;
        }
      }
    }
  }

  // ---- anticausal sweep up from min(g1 + K, H + K) - 1; outputs for g in [g0, g1)
  //      (the plane row, causal sums and f of the next row are loaded one step ahead)
  DrAnti as[NPG];
#pragma unroll
  for (int q = 0; q < NPG; q++) as[q].zero();
  unsigned nguard = 0;
  const int ge = min(g1 + K, H + K) - 1;
  float2 nx[NPG], ny[NPG];
  float nf = 0.f;
  auto fetch = [&](int g) {
    const long long o = prow(g);
#pragma unroll
    for (int q = 0; q < NPG; q++) {
      GC_CHK(p, pl + q * pstride + o, 8);
      nx[q] = __ldg(pl + q * pstride + o);
    }
    if (g < g1) {
      const long long oy = (long long)(g - p.out_row0) * p.Wd;
#pragma unroll
      for (int q = 0; q < NPG; q++) {
        GC_CHK(p, &ys[q * ys_pair + oy], 8);
        ny[q] = ys[q * ys_pair + oy];
      }
      GC_CHK(p, row_ptr(p, b, g) + xc, 4);
      nf = __ldg(row_ptr(p, b, g) + xc);
    }
  };
  fetch(ge);
#pragma unroll 1
  for (int g = ge; g >= g0; g--) {
    float2 cx[NPG], cy[NPG];
#pragma unroll
    for (int q = 0; q < NPG; q++) {
      cx[q] = nx[q];
      cy[q] = ny[q];
    }
    const float fo = nf;
    if (g - 1 >= g0) fetch(g - 1);
    if (g >= g1) {
#pragma unroll
      for (int q = 0; q < NPG; q++) as[q].step(p, cx[q]);
      continue;
    }
    const int yo = g - p.out_row0;
    const float a = p.raw ? 0.f : centre_a(p, fo);
    const float2 a2 = f2s(a * a);
    float2 pw = make_float2(1.f, a), P2 = make_float2(0.f, 0.f), Q2 = make_float2(0.f, 0.f);
    float vpy = 0.f, raw0 = 0.f;
#pragma unroll
    for (int q = 0; q < NPG; q++) {
      const float2 F = f2add(as[q].step(p, cx[q]), cy[q]);   // Fbar'_{2q}, Fbar'_{2q+1}
      if (q == 0) raw0 = F.x;
      // eqs. (8)-(9): Q += chat_n a'^n Fbar_n, P += chat_n a'^n Fbar_{n+1}
      const float2 v2 = f2mul(p.chat2[q], pw);
      Q2 = f2fma(v2, F, Q2);
      P2 = f2fma(make_float2(vpy, v2.x), F, P2);
      vpy = v2.y;
      pw = f2mul(pw, a2);
    }
    if (xok) {
      const float Q = Q2.x + Q2.y, P = P2.x + P2.y;
      float o;
      if (p.raw) {
        o = raw0;
      } else if (Q > 0.f && isfinite(Q) && isfinite(P)) {
        o = p.t_c + p.t_h * __fdividef(P, Q);          // eq. (10) + uncentring
      } else {                                          // guard (R8)
        o = fminf(fmaxf(fo, p.L), p.U);
        nguard++;
      }
      GC_CHK(p, &p.out[b * p.out_img_stride + (long long)yo * p.Wd + x], 4);
      p.out[b * p.out_img_stride + (long long)yo * p.Wd + x] = o;
    }
  }
  count_guarded(p.fallback, 0xffffffffu, nguard);
}

// ------------------------------------------------------------------ dispatch

namespace {

template <typename K>
long long dr_resident_warps(K kern, size_t smem, int num_sms) {
  int blocks = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, kern, 32 * kDrWarps, smem) != cudaSuccess) blocks = 1;
  return (long long)std::max(1, blocks) * kDrWarps * num_sms;
}

template <int NPG>
cudaError_t launch_dr(const KParams& p0, cudaStream_t s) {
  const size_t smem_r = (size_t)kDrWarps * sizeof(DrRowSmem);
  static std::atomic<unsigned long long> ready{0};
  static std::atomic<long long> res_r{1}, res_c{1};
  cudaError_t e = once_per_device(ready, [&]() {
    cudaError_t r = cudaFuncSetAttribute(k_row_dr<NPG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_r);
    if (r == cudaSuccess) {
      res_r.store(dr_resident_warps(k_row_dr<NPG>, smem_r, p0.num_sms));
      res_c.store(dr_resident_warps(k_col_dr<NPG>, 0, p0.num_sms));
    }
    return r;
  });
  if (e != cudaSuccess) return e;
  // segments: lead-in K per sweep direction; row-pass segments are multiples of the 8-column chunk
  KParams p = p0;
  pick_segments(p.Wd, (long long)((p.in_rows + 31) / 32) * p.B, p.dr_K, res_r.load(), kDrChunk, p.dr_seg_x,
                p.dr_nseg_x);
  pick_segments(p.out_rows, (long long)((p.Wd + 31) / 32) * p.B, p.dr_K, res_c.load(), 1, p.dr_seg_y, p.dr_nseg_y);
  const long long ntr = (long long)((p.in_rows + 31) / 32) * p.dr_nseg_x * p.B;
  const long long ntc = (long long)((p.Wd + 31) / 32) * p.dr_nseg_y * p.B;
  if (p.ev[0]) cudaEventRecord(p.ev[0], s);
  k_row_dr<NPG><<<(unsigned)((ntr + kDrWarps - 1) / kDrWarps), 32 * kDrWarps, smem_r, s>>>(p);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (p.ev[1]) cudaEventRecord(p.ev[1], s);
  e = launch_k(k_col_dr<NPG>, dim3((unsigned)((ntc + kDrWarps - 1) / kDrWarps)), dim3(32 * kDrWarps), 0, s,
               p.ev[1] == nullptr, p);
  if (p.ev[2]) cudaEventRecord(p.ev[2], s);
  return e;
}

}  // namespace

cudaError_t launch_deriche_two_pass(const KParams& p, cudaStream_t s) {
  switch (p.NP) {
    case 1: return launch_dr<1>(p, s);
    case 2: return launch_dr<2>(p, s);
    case 3: return launch_dr<3>(p, s);
    case 4: return launch_dr<4>(p, s);
    case 5: return launch_dr<5>(p, s);
    case 6: return launch_dr<6>(p, s);
    case 7: return launch_dr<7>(p, s);
    case 8: return launch_dr<8>(p, s);
    default: return cudaErrorInvalidValue;   // N > 14: rejected by gc_api.cpp (GC_ERANGE)
  }
}

}  // namespace gc
