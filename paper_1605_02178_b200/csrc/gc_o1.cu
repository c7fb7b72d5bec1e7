// gc_o1.cu — O(1)-per-pixel evaluation of eq. (7) for the GCF hot path on sm_100a.
//
// Eq. (7) sums the N+2 auxiliary planes over the truncated window Omega = [-W, W]^2 with
// sampled Gaussian taps.  The paper reaches O(1) cost per pixel "using separability
// and recursion" with Deriche's untruncated IIR; this build keeps eq. (7)'s
// truncated window as the definition (R3) and reaches O(1) with an EXACT-WINDOW
// recursion instead:
//
//   k_m ~= sum_{q=0}^{K-1} alpha_q cos(w_q m),   |m| <= W    (host fit, gc_operator.cpp: K = 5,
//                                                             w_0 = 0 and four optimised frequencies,
//                                                             max error ~5e-8 of the peak tap)
//   S_q(i) = sum_{m=-W}^{W} cos(w_q m) x(i+m)                 (window sum, exactly W wide)
//   S_q(i+1) - 2 cos(w_q) S_q(i) + S_q(i-1)
//        = cos(w_q W) [x(i+W+1) + x(i-W-1)] - cos(w_q (W+1)) [x(i+W) + x(i-W)]
//
// evaluated in Reinsch's form (D = S(i) - S(i-1); D += -4 sin^2(w/2) S + input; S += D),
// which keeps the fp32 rounding of the unit-circle resonator small for small w_q (all four
// w_q W / pi lie in 0.87..3.80).  q = 0 is the plain box sum S_0(i+1) = S_0(i) + x(i+W+1) -
// x(i-W).  The weights alpha_q are folded into the states, so the filtered value is their sum.
// Each line segment starts from a zero state 2W+1 samples early ("lead-in"), so no state crosses
// segment or task boundaries and the result is a pure function of the window — the same
// truncated sum as eq. (7), up to the fit error and fp32 rounding.  Per plane pair and sample:
// 24 packed FP32x2 instructions, independent of sigma_s.
//
//   k_row_o1 (a1 + a2, horizontal): warp = 32 image rows (lane = row) x one x-segment x
//            <= 4 plane pairs; f is staged through a transposed shared-memory tile (coalesced
//            128-byte row loads), the planes F'_n of eq. (6) are generated in registers for
//            the entering and leaving samples, and the filtered pairs are transposed back
//            through shared memory for 128-byte row stores.  Output layout as the FIR path:
//            [B][NP][in_rows][Wd] float2.
//   k_col_o1 (a2 vertical + a3): warp = 32/G columns x G plane-pair groups (lane = column),
//            walking down one y-segment; loads of the entering/leaving rows are coalesced and
//            prefetched one step ahead; partial P', Q' of eqs. (8)-(9) are reduced across the
//            G groups with shuffles; eq. (10) and the guard (R8) as in gc_fir.cu.
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "gc_device.cuh"

namespace gc {

constexpr int kO1Warps = 4;     // warps per CTA (independent tasks)
constexpr int kO1CH = 16;       // positions per staged chunk
constexpr int kO1TS = 17;       // staged tile row stride (float2): 2 wavefronts per warp access
constexpr int kO1OC = 4;        // output positions per store chunk (= main-loop unroll)
constexpr int kO1RowNPG = 4;    // plane pairs per row-pass warp (max)
constexpr int kO1OS = 36;       // out tile position stride (float2): conflict-free 64-bit reads
constexpr int kO1RS = 20;       // raw f row stride (floats): 16-byte cp.async rows, LDS.128 conflict-free

struct RowO1Smem {
  float2 fin[32 * kO1TS];                  // entering stream  [row][pos] = (e a'^{2p0}, a')
  float2 fout[32 * kO1TS];                 // leaving stream   [row][pos]
  float2 o[kO1RowNPG][kO1OC][kO1OS];       // filtered pairs   [pair][pos][row]
  float raw[2][32 * kO1RS];                // f of the NEXT chunk of each stream (cp.async prefetch)
};

// L2 cache policies (createpolicy): streaming data that is not read again in this kernel (plane
// stores of the row pass, the output) is marked evict_first so it does not push out what is
// (f, re-read by the leaving stream and the other pair group; the column pass's window rows).
__device__ __forceinline__ unsigned long long l2_evict_first() {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ unsigned long long l2_evict_last() {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void st_f2_hint(float2* a, float2 v, unsigned long long pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v2.f32 [%0], {%1, %2}, %3;" ::"l"(a), "f"(v.x), "f"(v.y),
               "l"(pol)
               : "memory");
}
__device__ __forceinline__ void st_f_hint(float* a, float v, unsigned long long pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(a), "f"(v), "l"(pol) : "memory");
}

// Prefetch f of this lane's row at the 16 positions [pc, pc+16) (whole-sample mirroring in x)
// into raw (one cp.async group per call): the stage one chunk later finds it in shared memory
// instead of stalling on DRAM (ncu r01: long_scoreboard was the top stall of k_row_o1).
__device__ __forceinline__ void o1_prefetch_row(const KParams& p, float* raw, const float* rowp, int pc, int lane,
                                               bool vec) {
  float* d = raw + lane * kO1RS;
  const unsigned s = (unsigned)__cvta_generic_to_shared(d);
  if (vec && pc >= 0 && pc + kO1CH <= p.Wd) {
#pragma unroll
    for (int k = 0; k < kO1CH / 4; k++)
    {
      GC_CHK(p, rowp + pc + 4 * k, 16);
      asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(s + 16 * k),
                   "l"(rowp + pc + 4 * k), "l"(l2_evict_last())
                   : "memory");
    }
  } else {
#pragma unroll 1
    for (int k = 0; k < kO1CH; k++)
    {
      GC_CHK(p, rowp + mirror(pc + k, p.Wd), 4);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s + 4 * k), "l"(rowp + mirror(pc + k, p.Wd))
                   : "memory");
    }
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

// Stage this lane's row at the 16 positions of the aligned chunk [pc, pc+16) (whole-sample
// mirroring in x) as v = (F'_{2p0}, a') = (e a'^{2p0}, a') of eq. (6), or (f, 0) for
// gc_gaussian; then F'_{2p0+1} = v.x v.y and the pair step is a'^2 = v.y^2.
// (f comes from the prefetch buffer `raw`, whose cp.async group the caller has waited for; the
// next chunk of the same stream is prefetched into it afterwards)
// (inlined: as a call, the ABI saves the caller's ~100 live state registers around it — measured
// 8.2 instead of 6.0 ms for the c5 row pass)
// PM = plane-generation mode, a template parameter so that each row-pass instantiation carries one
// staging variant (four inlined sites per task; ncu r02: no_instruction stalls): 0 = gc_gaussian
// (f, 0), 1 = first pair group (p0 = 0), 2 = p0 = 4, 3 = any p0.
enum { kPmRaw = 0, kPm0 = 1, kPm4 = 2, kPmAny = 3 };

template <int WAIT, int PM>
__device__ __forceinline__ void o1_stage_row(const KParams& p, float2* t, float* raw, const float* rowp, int pc,
                                            int lane, bool vec, int p0) {
  asm volatile("cp.async.wait_group %0;" ::"n"(WAIT) : "memory");
  float v[kO1CH];
  {
    const float4* r4 = reinterpret_cast<const float4*>(raw + lane * kO1RS);
#pragma unroll
    for (int k = 0; k < kO1CH / 4; k++) {
      const float4 u = r4[k];
      v[4 * k] = u.x; v[4 * k + 1] = u.y; v[4 * k + 2] = u.z; v[4 * k + 3] = u.w;
    }
  }
  float2* d = t + lane * kO1TS;
  __syncwarp();
  if constexpr (PM == kPmRaw) {
#pragma unroll
    for (int k = 0; k < kO1CH; k++) d[k] = make_float2(v[k], 0.f);
  } else if constexpr (PM == kPm0) {
#pragma unroll
    for (int k = 0; k < kO1CH; k++) {
      float a, e;
      centre(p, v[k], a, e);
      d[k] = make_float2(e, a);
    }
  } else if constexpr (PM == kPm4) {
#pragma unroll
    for (int k = 0; k < kO1CH; k++) {
      float a, e;
      centre(p, v[k], a, e);
      const float a2 = a * a, a4 = a2 * a2;
      d[k] = make_float2(e * (a4 * a4), a);
    }
  } else {
#pragma unroll
    for (int k = 0; k < kO1CH; k++) {
      float a, e;
      centre(p, v[k], a, e);
      float pw = 1.f, base = a * a;
      for (int kk = p0; kk; kk >>= 1) {
        if (kk & 1) pw *= base;
        base *= base;
      }
      d[k] = make_float2(e * pw, a);
    }
  }
  // this stream's next chunk, issued after v has been consumed (the copy overwrites raw)
  o1_prefetch_row(p, raw, rowp, pc + kO1CH, lane, vec);
  __syncwarp();
}

// One step of the exact-window recursion for one plane pair (Reinsch form).
//   A = x(i+W+1) + x(i-W-1), B = x(i+W) + x(i-W), box: S0 += x(i+W+1) - x(i-W)
// The fit weights alpha_q are folded into the state (S'_q = alpha_q S_q, a linear recursion with
// inputs scaled by alpha_q: o1_a / o1_nb carry alpha_q, the box input alpha_0), so the filtered
// value is the plain sum of the states (a 3-deep add tree instead of a 6-deep FMA chain).
// The state-only FMA comes first: the input samples A, B (shared-memory loads) arrive last.
__device__ __forceinline__ void o1_update(const KParams& p, float2& S0, float2* S, float2* D, float2 A, float2 B,
                                          float2 xin, float2 xout) {
  S0 = f2fma(f2s(p.o1_alpha[0]), f2sub(xin, xout), S0);
  // (written stage by stage across the resonators: consecutive instructions are independent)
  float2 d[kO1K - 1];
#pragma unroll
  for (int t = 0; t < kO1K - 1; t++) d[t] = f2fma(f2s(p.o1_nk[t + 1]), S[t], D[t]);
#pragma unroll
  for (int t = 0; t < kO1K - 1; t++) d[t] = f2fma(f2s(p.o1_a[t + 1]), A, d[t]);
#pragma unroll
  for (int t = 0; t < kO1K - 1; t++) {
    d[t] = f2fma(f2s(p.o1_nb[t + 1]), B, d[t]);
    D[t] = d[t];
    S[t] = f2add(S[t], d[t]);
  }
}

__device__ __forceinline__ float2 o1_output(const KParams& p, float2 S0, const float2* S) {
  static_assert(kO1K == 5, "o1_output's add tree assumes the box + 4 resonators");
  return f2add(f2add(S0, S[0]), f2add(f2add(S[1], S[2]), S[3]));
}

template <int NPG>
struct RowO1State {
  float2 S0[NPG], S[NPG][kO1K - 1], D[NPG][kO1K - 1], Ep[NPG], Lp[NPG];
};

// One output step at x (window centred on x), output slot j of the current store chunk.
template <int NPG, int PM>
__device__ __forceinline__ void row_o1_step(const KParams& p, RowO1Smem& sm, RowO1State<NPG>& st, int x, int j,
                                            const float* rowp, bool vec, int p0, int lane) {
  const int R = p.R;
  const int pe_pos = x + R + 1, pl_pos = x - R;
  // the two streams stage on different steps ((2W+1) is odd), so the newest cp.async group is
  // always the other stream's prefetch: wait_group 1 finds this stream's chunk complete
  if ((pe_pos & (kO1CH - 1)) == 0) o1_stage_row<1, PM>(p, sm.fin, sm.raw[0], rowp, pe_pos, lane, vec, p0);
  if ((pl_pos & (kO1CH - 1)) == 0) o1_stage_row<1, PM>(p, sm.fout, sm.raw[1], rowp, pl_pos, lane, vec, p0);
  const float2 ve = sm.fin[lane * kO1TS + (pe_pos & (kO1CH - 1))];
  const float2 vl = sm.fout[lane * kO1TS + (pl_pos & (kO1CH - 1))];
  const float a2e = ve.y * ve.y, a2l = vl.y * vl.y;
#ifndef GC_ROW_STAGED
#define GC_ROW_STAGED 1
#endif
#if GC_ROW_STAGED
  // The NPG pairs' updates interleaved by stage (all pairs' first FMA, then all second FMAs, ...):
  // consecutive instructions are independent, so a warp can issue back to back instead of waiting
  // on each resonator's 4-deep dependency chain (ncu r02: 'wait' was k_row_o1's top stall).
  float2 pe[NPG], pl[NPG];
  pe[0] = make_float2(ve.x, ve.x * ve.y);
  pl[0] = make_float2(vl.x, vl.x * vl.y);
#pragma unroll
  for (int q = 1; q < NPG; q++) {
    pe[q] = f2mul(pe[q - 1], f2s(a2e));
    pl[q] = f2mul(pl[q - 1], f2s(a2l));
  }
#pragma unroll
  for (int q = 0; q < NPG; q++) sm.o[q][j][lane] = o1_output(p, st.S0[q], st.S[q]);
  float2 A[NPG], B[NPG], d[NPG][kO1K - 1];
#pragma unroll
  for (int q = 0; q < NPG; q++) {
    A[q] = f2add(pe[q], st.Lp[q]);
    B[q] = f2add(st.Ep[q], pl[q]);
    st.S0[q] = f2fma(f2s(p.o1_alpha[0]), f2sub(pe[q], pl[q]), st.S0[q]);
  }
#pragma unroll
  for (int t = 0; t < kO1K - 1; t++)
#pragma unroll
    for (int q = 0; q < NPG; q++) d[q][t] = f2fma(f2s(p.o1_nk[t + 1]), st.S[q][t], st.D[q][t]);
#pragma unroll
  for (int t = 0; t < kO1K - 1; t++)
#pragma unroll
    for (int q = 0; q < NPG; q++) d[q][t] = f2fma(f2s(p.o1_a[t + 1]), A[q], d[q][t]);
#pragma unroll
  for (int t = 0; t < kO1K - 1; t++)
#pragma unroll
    for (int q = 0; q < NPG; q++) {
      d[q][t] = f2fma(f2s(p.o1_nb[t + 1]), B[q], d[q][t]);
      st.D[q][t] = d[q][t];
      st.S[q][t] = f2add(st.S[q][t], d[q][t]);
    }
#pragma unroll
  for (int q = 0; q < NPG; q++) {
    st.Ep[q] = pe[q];
    st.Lp[q] = pl[q];
  }
#else
  float2 pe = make_float2(ve.x, ve.x * ve.y), pl = make_float2(vl.x, vl.x * vl.y);
#pragma unroll
  for (int q = 0; q < NPG; q++) {
    sm.o[q][j][lane] = o1_output(p, st.S0[q], st.S[q]);
    o1_update(p, st.S0[q], st.S[q], st.D[q], f2add(pe, st.Lp[q]), f2add(st.Ep[q], pl), pe, pl);
    st.Ep[q] = pe;
    st.Lp[q] = pl;
    pe = f2mul(pe, f2s(a2e));
    pl = f2mul(pl, f2s(a2l));
  }
#endif
}

template <int NPG, int PM>
__device__ __forceinline__ void row_o1_task(const KParams& p, RowO1Smem& sm, int b, int r0, int xs, int xe, int p0,
                                            int lane) {
  const int R = p.R;
  const int lead = 2 * R + 1;        // lead-in: zero state, empty window, 2W+1 entering samples
  const int P0 = xs - R;             // first position of both streams
  RowO1State<NPG> st;
#pragma unroll
  for (int q = 0; q < NPG; q++) {
    st.S0[q] = st.Ep[q] = st.Lp[q] = make_float2(0.f, 0.f);
#pragma unroll
    for (int t = 0; t < kO1K - 1; t++) st.S[q][t] = st.D[q][t] = make_float2(0.f, 0.f);
  }
  const float* rowp = row_ptr(p, b, p.in_row0 + min(r0 + lane, p.in_rows - 1));
  const bool vec = ((p.Wd & 3) == 0) && ((reinterpret_cast<uintptr_t>(rowp) & 15) == 0);

  // ---- lead-in: the state at the first output x = xs from the 2W+1 samples of its window
  o1_prefetch_row(p, sm.raw[0], rowp, P0 & ~(kO1CH - 1), lane, vec);
  o1_prefetch_row(p, sm.raw[1], rowp, (xs - R) & ~(kO1CH - 1), lane, vec);
  const float4* const lt = p.o1_lead;
  // chunk by chunk (one staging per chunk), the samples of a chunk unrolled: their latency
  // chains (shared-memory load, the a^2 power chain across the pairs) overlap
#pragma unroll 1
  for (int s0 = 0; s0 < lead;) {
    const int pos0 = P0 + s0;
    // (only this stream stages here: wait for all groups)
    o1_stage_row<0, PM>(p, sm.fin, sm.raw[0], rowp, pos0 & ~(kO1CH - 1), lane, vec, p0);
    const int n = min(kO1CH - (pos0 & (kO1CH - 1)), lead - s0);
    if (lt) {
      // direct: S_q(xs) and D_q(xs) = S_q(xs) - S_q(xs-1) as dot products with the fitted taps
      // (the state the recursion reaches from a zero state after these 2W+1 steps, with 9
      // instead of 17 packed operations per pair and sample)
#pragma unroll 4
      for (int i = 0; i < n; i++) {
        const int s = s0 + i;
        const float2 ve = sm.fin[lane * kO1TS + ((pos0 + i) & (kO1CH - 1))];
        float2 pe = make_float2(ve.x, ve.x * ve.y);
        const float a2e = ve.y * ve.y;
        GC_CHK(p, &lt[2 * s], 32);
        const float4 c = __ldg(&lt[2 * s]), d = __ldg(&lt[2 * s + 1]);
        const float cq[4] = {c.x, c.y, c.z, c.w}, dq[4] = {d.x, d.y, d.z, d.w};
#pragma unroll
        for (int q = 0; q < NPG; q++) {
          st.S0[q] = f2fma(f2s(p.o1_alpha[0]), pe, st.S0[q]);
#pragma unroll
          for (int t = 0; t < kO1K - 1; t++) {
            st.S[q][t] = f2fma(f2s(cq[t]), pe, st.S[q][t]);
            st.D[q][t] = f2fma(f2s(dq[t]), pe, st.D[q][t]);
          }
          st.Ep[q] = pe;
          pe = f2mul(pe, f2s(a2e));
        }
      }
    } else {
      // recursion from a zero state over windows xs-2W-1 .. xs-1 (leaving samples still zero)
#pragma unroll 1
      for (int i = 0; i < n; i++) {
        const float2 ve = sm.fin[lane * kO1TS + ((pos0 + i) & (kO1CH - 1))];
        float2 pe = make_float2(ve.x, ve.x * ve.y);
        const float a2e = ve.y * ve.y;
#pragma unroll
        for (int q = 0; q < NPG; q++) {
          o1_update(p, st.S0[q], st.S[q], st.D[q], pe, st.Ep[q], pe, make_float2(0.f, 0.f));
          st.Ep[q] = pe;
          pe = f2mul(pe, f2s(a2e));
        }
      }
    }
    s0 += n;
  }
  // ---- outputs x = xs .. xe-1, in chunks of kO1OC positions (xs is a multiple of 32).  The
  // leaving stream's first chunk: staged here unless x = xs itself starts a chunk (then the first
  // step stages it; staging it twice would read the prefetch of the chunk after it)
  if ((xs - R) & (kO1CH - 1)) o1_stage_row<0, PM>(p, sm.fout, sm.raw[1], rowp, (xs - R) & ~(kO1CH - 1), lane, vec, p0);
  // row_o1_step stages with wait_group 1, which assumes the newest cp.async group is the OTHER
  // stream's prefetch.  After the staging above the only group in flight is the leaving stream's
  // own prefetch, and for R mod 16 in 1..7 the leaving stream stages again before the entering
  // stream does: wait_group 1 would let it read raw[1] before that prefetch landed (stale samples,
  // a timing-dependent error in the window sum).  An empty group restores the invariant.
  asm volatile("cp.async.commit_group;" ::: "memory");
  // O(1) plane layout [B][rows][NP][Wd]: the NP pairs of one image row are adjacent rows of
  // a 2-D [B*rows*NP][Wd] tensor, so the column pass fetches a row's pairs with one TMA box
  const long long rstride = (long long)p.NP * p.Wd;         // float2 between image rows
  constexpr int ORS = 32 / kO1OC;                           // rows per store instruction
  const int orow = lane / kO1OC, ocol = lane % kO1OC;
  const int rows_left = p.in_rows - (r0 + orow);            // rows r0+orow+ORS j valid for ORS j < rows_left
  float2* const obase = p.planes + b * p.planes_img_stride + (long long)(r0 + orow) * rstride +
                        (long long)p0 * p.Wd + ocol;
  const unsigned long long pol_stream = l2_evict_first();
#pragma unroll 1
  for (int x = xs; x < xe; x += kO1OC) {
    const int nb = min(kO1OC, xe - x);
#pragma unroll 1
    for (int j = 0; j < nb; j++) row_o1_step<NPG, PM>(p, sm, st, x + j, j, rowp, vec, p0, lane);
    // store the chunk: per pair, kO1OC positions x 32 rows (ORS rows x 8 kO1OC bytes per instruction)
    __syncwarp();
    if (ocol < nb) {
      float2* o = obase + x;
#pragma unroll
      for (int q = 0; q < NPG; q++) {
#pragma unroll
        for (int j = 0; j < 32 / ORS; j++)
          if (ORS * j < rows_left) {
            GC_CHK(p, &o[(long long)(ORS * j) * rstride], 8);
            st_f2_hint(&o[(long long)(ORS * j) * rstride], sm.o[q][ocol][ORS * j + orow], pol_stream);
          }
        o += p.Wd;
      }
    }
    __syncwarp();
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");      // no copy may land after the task
}

// Task decode of the row pass: groups of kO1RowNPG plane pairs and one remainder group last,
// tasks numbered group-major so that the dynamic fetch runs every task of the full groups before
// the smaller one (longest-processing-time-first: the tail is short tasks).  (Measured slower:
// balanced groups, NP = 6 as 3 + 3 instead of 4 + 2, r02ai; the groups of one segment adjacent
// so that they share f in L2, r02ap: c5 row 4.78 -> 5.01 ms.)
struct RowO1Task {
  int b, rb, sx, p0, npl;
};
__device__ __forceinline__ RowO1Task row_o1_decode(const KParams& p, int task, int nrb) {
  const int per_group = nrb * p.o1_nseg_x * p.B;
  const int g = task / per_group, rest = task - g * per_group;
  RowO1Task t;
  t.sx = rest % p.o1_nseg_x;
  t.rb = (rest / p.o1_nseg_x) % nrb;
  t.b = rest / (p.o1_nseg_x * nrb);
  t.p0 = g * kO1RowNPG;
  t.npl = min(kO1RowNPG, p.NP - t.p0);
  return t;
}

// Persistent: one CTA per resident slot, each warp fetching tasks (32 rows x one x-segment x one
// plane-pair group) from a counter that the launch zeroes, until none is left.
__global__ void __launch_bounds__(32 * kO1Warps, 3) k_row_o1(const KParams p, unsigned* task_ctr) {
  extern __shared__ float4 smem_o1r[];
  pdl_trigger();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  RowO1Smem& sm = reinterpret_cast<RowO1Smem*>(smem_o1r)[warp];
  const int nrb = (p.in_rows + 31) / 32;
  const int ntask = nrb * p.o1_nseg_x * p.o1_groups * p.B;
#pragma unroll 1
  for (;;) {
    int task = 0;
    if (lane == 0) task = (int)atomicAdd(task_ctr, 1u);
    task = __shfl_sync(0xffffffffu, task, 0);
    if (task >= ntask) break;
    const RowO1Task t = row_o1_decode(p, task, nrb);
    const int xs = t.sx * p.o1_seg_x, xe = min(xs + p.o1_seg_x, p.Wd);
    if (p.raw) {                                   // gc_gaussian: one pair (f, 0)
      row_o1_task<1, kPmRaw>(p, sm, t.b, t.rb * 32, xs, xe, 0, lane);
      continue;
    }
    auto go = [&](auto pm) {
      constexpr int PM = decltype(pm)::value;
      switch (t.npl) {
        case 1: row_o1_task<1, PM>(p, sm, t.b, t.rb * 32, xs, xe, t.p0, lane); break;
        case 2: row_o1_task<2, PM>(p, sm, t.b, t.rb * 32, xs, xe, t.p0, lane); break;
        case 3: row_o1_task<3, PM>(p, sm, t.b, t.rb * 32, xs, xe, t.p0, lane); break;
        default: row_o1_task<4, PM>(p, sm, t.b, t.rb * 32, xs, xe, t.p0, lane); break;
      }
    };
    if (t.p0 == 0) go(std::integral_constant<int, kPm0>());
    else if (t.p0 == 4) go(std::integral_constant<int, kPm4>());
    else go(std::integral_constant<int, kPmAny>());
  }
}

// ------------------------------------------------------------------ column pass + eqs. (8)-(10)

constexpr int kO1D = 4;          // column pass: cp.async pipeline depth (rows in flight)
constexpr int kO1ColNPGMax = 7;

struct alignas(128) ColO1Smem {   // 128-byte aligned: TMA destinations
  float2 ring[kO1D][2][kO1ColNPGMax][32];   // [stage][enter/leave][pair][lane]
  float fring[kO1D][32];                    // f at the output row
  unsigned long long full[kO1D];            // TMA mode: one mbarrier per stage
};

__device__ __forceinline__ void o1_mbar_init(unsigned long long* bar) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s));
}
__device__ __forceinline__ void o1_mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s), "r"(bytes) : "memory");
}
__device__ __forceinline__ void o1_mbar_wait(unsigned long long* bar, unsigned phase) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(s),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void o1_tma_2d(void* smem, const CUtensorMap* map, int c0, int c1, unsigned long long* bar) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(s),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(b)
      : "memory");
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// TMA = true (G = 1, NP <= NPG): each step's entering and leaving rows arrive as two 2-D TMA
// boxes of [NP pairs][32 columns] (one elected lane, mbarrier per stage); otherwise per-lane
// 8-byte cp.async copies.
template <int NPG, int G, bool TMA>
__global__ void __launch_bounds__(32 * kO1Warps) k_col_o1(const __grid_constant__ CUtensorMap tmap, const KParams p) {
  constexpr int CW = 32 / G;                       // columns per warp
  extern __shared__ __align__(1024) float4 smem_o1c[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  ColO1Smem& sm = reinterpret_cast<ColO1Smem*>(smem_o1c)[warp];
  const int ncb = (p.Wd + CW - 1) / CW;
  const int ntask = ncb * p.o1_nseg_y * p.B;
  const int task = blockIdx.x * kO1Warps + warp;
  if (task >= ntask) return;
  const int cb = task % ncb;
  const int sy = (task / ncb) % p.o1_nseg_y;
  const int b = task / (ncb * p.o1_nseg_y);
  const int g = lane / CW;
  const int x = cb * CW + (lane % CW);
  const bool xok = x < p.Wd;
  const int xc = xok ? x : p.Wd - 1;
  const int ys = sy * p.o1_seg_y, ye = min(ys + p.o1_seg_y, p.out_rows);
  const int R = p.R;
  const int lead = 2 * R + 1;
  const int p0 = g * NPG;
  const long long rstride = (long long)p.NP * p.Wd;          // layout [B][rows][NP][Wd]
  const float2* const src = p.planes + b * p.planes_img_stride + (long long)p0 * p.Wd + xc;
  int npl = p.NP - p0;                              // valid pairs of this lane's group
  npl = npl < 0 ? 0 : (npl > NPG ? NPG : npl);

  float2 cq[NPG];
#pragma unroll
  for (int q = 0; q < NPG; q++) cq[q] = (p0 + q < kMaxPairs) ? p.chat2[p0 + q] : make_float2(0.f, 0.f);
  const float cprev = p0 > 0 ? p.chat2[p0 - 1].y : 0.f;   // chat_{2 p0 - 1}

  float2 S0[NPG], S[NPG][kO1K - 1], D[NPG][kO1K - 1], Ep[NPG], Lp[NPG];
#pragma unroll
  for (int q = 0; q < NPG; q++) {
    S0[q] = Ep[q] = Lp[q] = make_float2(0.f, 0.f);
#pragma unroll
    for (int t = 0; t < kO1K - 1; t++) S[q][t] = D[q][t] = make_float2(0.f, 0.f);
  }
  // padding pairs (p0 + q >= NP) read zeros: their ring entries are never written
#pragma unroll
  for (int st = 0; st < kO1D; st++)
#pragma unroll
    for (int q = 0; q < NPG; q++)
      if (q >= npl) sm.ring[st][0][q][lane] = sm.ring[st][1][q][lane] = make_float2(0.f, 0.f);

  if (TMA) {
    if (lane == 0) {
      for (int st = 0; st < kO1D; st++) o1_mbar_init(&sm.full[st]);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
  }
  pdl_wait();                                       // planes from k_row_o1
  const bool fseg = p.seg[0].rows > 0 && p.out_row0 >= p.seg[0].row0 &&
                    p.out_row0 + p.out_rows <= p.seg[0].row0 + p.seg[0].rows;
  const float* const frow = p.seg[0].ptr + b * p.seg_img_stride +
                            (long long)(p.out_row0 - p.seg[0].row0) * p.Wd + xc;
  // step i (window centred on output-relative row i): entering row i+R+1, leaving row i-R
  auto issue = [&](int i, int st) {
    // (the entering row of the last step feeds the window after ye, which is never output: at
    // the bottom of an interior window it lies one row past the plane buffer, so clamp it)
    const int ye_row = min(mirror(p.out_row0 + i + R + 1, p.H) - p.in_row0, p.in_rows - 1);
    // (during the lead-in the leaving sample is masked to zero; read a valid row instead)
    const int yl_row = i >= ys ? mirror(p.out_row0 + i - R, p.H) - p.in_row0 : ye_row;
    if (TMA) {
      if (lane == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // prior reads of the stage
        o1_mbar_expect_tx(&sm.full[st], 2u * p.NP * 32u * 8u);
        const int x0 = cb * CW;
        o1_tma_2d(&sm.ring[st][0][0][0], &tmap, x0, (b * p.in_rows + ye_row) * p.NP, &sm.full[st]);
        o1_tma_2d(&sm.ring[st][1][0][0], &tmap, x0, (b * p.in_rows + yl_row) * p.NP, &sm.full[st]);
      }
    } else {
      const long long re = (long long)ye_row * rstride, rl = (long long)yl_row * rstride;
#pragma unroll
      for (int q = 0; q < NPG; q++) {
        if (q < npl) {
          GC_CHK(p, src + q * p.Wd + re, 8);
          GC_CHK(p, src + q * p.Wd + rl, 8);
          cp_async8(&sm.ring[st][0][q][lane], src + q * p.Wd + re);
          cp_async8(&sm.ring[st][1][q][lane], src + q * p.Wd + rl);
        }
      }
    }
    const int fi = max(i, 0);
    GC_CHK(p, fseg ? frow + (long long)fi * p.Wd : row_ptr(p, b, p.out_row0 + fi) + xc, 4);
    cp_async4(&sm.fring[st][lane], fseg ? frow + (long long)fi * p.Wd : row_ptr(p, b, p.out_row0 + fi) + xc);
  };
  const int i0 = ys - lead;
#pragma unroll
  for (int k = 0; k < kO1D - 1; k++) {
    if (i0 + k < ye) issue(i0 + k, k);
    cp_commit();
  }
  float* const outp = p.out + b * p.out_img_stride + x;
  unsigned nguard = 0;                              // guarded outputs of this lane (R8)
#pragma unroll 1
  for (int i = i0; i < ye; i++) {
    const int k = i - i0;
    if (TMA) __syncwarp();                          // all lanes are done with stage (k-1) % D
    if (i + kO1D - 1 < ye) issue(i + kO1D - 1, (k + kO1D - 1) % kO1D);
    cp_commit();
    cp_wait<kO1D - 1>();                            // this lane's copies for step i landed
    const int st = k % kO1D;
    if (TMA) o1_mbar_wait(&sm.full[st], (k / kO1D) & 1);
    float2 pe[NPG], pl[NPG];
    const bool live = i >= ys;                      // lead-in: leaving samples are zero
#pragma unroll
    for (int q = 0; q < NPG; q++) {
      pe[q] = sm.ring[st][0][q][lane];
      pl[q] = live ? sm.ring[st][1][q][lane] : make_float2(0.f, 0.f);
    }
    if (live) {
      const float fo = sm.fring[st][lane];
      // filtered pairs at row i, partial P', Q' over this group's planes (eqs. 8-9)
      const float a = p.raw ? 0.f : centre_a(p, fo);
      const float a2 = a * a;
      float pwg = 1.f;                                // a'^{2 NPG}: one group's power step
#pragma unroll
      for (int kk = 0; kk < NPG; kk++) pwg *= a2;
      float pw = 1.f, pwprev = 1.f;                   // a'^{2 p0} = pwg^g; a'^{2 (p0 - NPG)}
#pragma unroll
      for (int kk = 1; kk < G; kk++) {
        pwprev = kk < g ? pwprev * pwg : pwprev;
        pw = kk <= g ? pw * pwg : pw;
      }
      float aodd = a;                                 // a'^{2 NPG - 1}
#pragma unroll
      for (int kk = 1; kk < NPG; kk++) aodd *= a2;
      float2 Q2 = make_float2(0.f, 0.f), P2 = make_float2(0.f, 0.f);
      float2 pw2 = make_float2(pw, pw * a);
      float vprev = cprev * (pwprev * aodd);          // chat_{2p0-1} a'^{2p0-1} (0 for g = 0)
      float out_raw = 0.f;
#pragma unroll
      for (int q = 0; q < NPG; q++) {
        const float2 y = o1_output(p, S0[q], S[q]);
        if (q == 0) out_raw = y.x;
        const float2 v = f2mul(cq[q], pw2);
        Q2 = f2fma(v, y, Q2);
        P2 = f2fma(make_float2(vprev, v.x), y, P2);
        vprev = v.y;
        pw2 = f2mul(pw2, f2s(a2));
      }
      float Q = Q2.x + Q2.y, P = P2.x + P2.y;
#pragma unroll
      for (int m = CW; m < 32; m <<= 1) {
        Q += __shfl_xor_sync(0xffffffffu, Q, m);
        P += __shfl_xor_sync(0xffffffffu, P, m);
      }
      if (g == 0 && xok) {
        float o;
        if (p.raw) {
          o = out_raw;
        } else if (Q > 0.f && isfinite(Q) && isfinite(P)) {
          o = p.t_c + p.t_h * __fdividef(P, Q);          // eq. (10) + uncentring
        } else {                                         // guard (R8)
          o = fminf(fmaxf(fo, p.L), p.U);
          nguard++;
        }
        GC_CHK(p, &outp[(long long)i * p.Wd], 4);
        outp[(long long)i * p.Wd] = o;
      }
    }
    // update to window i+1
#pragma unroll
    for (int q = 0; q < NPG; q++) {
      o1_update(p, S0[q], S[q], D[q], f2add(pe[q], Lp[q]), f2add(Ep[q], pl[q]), pe[q], pl[q]);
      Ep[q] = pe[q];
      Lp[q] = pl[q];
    }
  }
  cp_wait<0>();
  count_guarded(p.fallback, 0xffffffffu, nguard);
}

// ------------------------------------------------------------------ pair-parallel column pass
//
// k_col_o1p<NP> (NP <= 8 plane pairs, even width): CTA = one 32-column strip x one y-segment;
// warp q < NP runs the vertical recursion of plane pair q for the 32 columns (lane = column),
// warp NP is the TMA producer.  Each step's entering row i+W+1 and leaving row i-W arrive as
// two [NP pairs x 32 columns] TMA boxes into a kPD-stage ring (mbarrier full/empty per stage);
// the consumers write their filtered pair of every output row into a [NP rows x NP pairs x 32]
// shared tile and, every NP rows, each warp folds one row's NP pairs into P', Q' (eqs. 8-9)
// and eq. (10).  Against k_col_o1 (one lane holds all NP pairs of its column): 1/NP of the
// recursion state per thread (~60 instead of 254 registers), NP x the warps per column strip,
// and — the point — a CTA's window of leaving rows is NP x 32 x (2W+1) x 8 B (174 KB at c5)
// with only kO1PCtas CTAs per SM, so the whole GPU's in-flight windows (~51 MB at 2 CTAs/SM)
// stay in L2 and the leaving rows are not re-read from HBM (k_col_o1 at c5: ~1200 resident
// warps x 174 KB = 206 MB, 123 B/px of DRAM traffic instead of 64; profiles/r01_ncu_full_o1_c5.txt).

constexpr int kPDMax = 48;       // ring stages (at most)
constexpr int kRPS = 4;          // image rows per ring stage: one [4 NP x 32] TMA box per direction in the
                                 // interior (per-row boxes where the rows are mirrored or clamped)

// Shared memory: this head, then the ring of nst stages, each = kRPS entering rows followed by
// kRPS leaving rows, a row = [NP pairs x 32 columns] float2.
#ifndef GC_COLP_TILES
#define GC_COLP_TILES 3
#endif
constexpr int kColT = GC_COLP_TILES;   // fold tile buffers: a warp runs up to kColT - 1 blocks ahead
#ifndef GC_COLP_STAGE_BLOCKS
#define GC_COLP_STAGE_BLOCKS 1
#endif
// rows per fold block: one ring stage (kRPS rows, the fold rotating over the warps), or NP rows
// (every warp folds one row of every block; the stage position is then a runtime counter)
template <int NP>
constexpr int colp_block_rows() { return GC_COLP_STAGE_BLOCKS ? kRPS : NP; }
template <int NP>
struct alignas(1024) ColPSmem {
  unsigned long long full[kPDMax], empty[kPDMax];
  unsigned long long tile_full[kColT], tile_free[kColT];   // per tile buffer: all NP warps wrote / folded it
  float2 tile[kColT][colp_block_rows<NP>()][NP][32];       // [buffer][row in block][pair][column]
};
template <int NP>
__host__ __device__ constexpr size_t colp_head() { return (sizeof(ColPSmem<NP>) + 1023) / 1024 * 1024; }
template <int NP>
__host__ __device__ constexpr size_t colp_stage() { return 2u * kRPS * NP * 32u * sizeof(float2); }

__device__ __forceinline__ void o1_mbar_init_n(unsigned long long* bar, unsigned n) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s), "r"(n));
}
__device__ __forceinline__ void o1_mbar_arrive(unsigned long long* bar) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s) : "memory");
}
__device__ __forceinline__ void o1_mbar_arrive_u32(unsigned s) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s) : "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_wait_u32(unsigned bar, unsigned phase) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(phase)
      : "memory");
}
#ifndef GC_COLP_BACKOFF_NS
#define GC_COLP_BACKOFF_NS 128
#endif
__device__ __forceinline__ void mbar_wait_backoff(unsigned bar, unsigned phase) {
  for (;;) {
    unsigned ok;
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
        "selp.u32 %0, 1, 0, P1;\n"
        "}\n"
        : "=r"(ok)
        : "r"(bar), "r"(phase)
        : "memory");
    if (ok) return;
    __nanosleep(GC_COLP_BACKOFF_NS);
  }
}
__device__ __forceinline__ float2 lds64(unsigned a) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sts64(unsigned a, float2 v) {
  asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(a), "f"(v.x), "f"(v.y) : "memory");
}
__device__ __forceinline__ void tma_2d_u32(unsigned dst, const CUtensorMap* map, int c0, int c1, unsigned bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
// 2-D TMA load with an L2 cache-policy hint (createpolicy descriptor)
__device__ __forceinline__ void tma_2d_hint(unsigned dst, const CUtensorMap* map, int c0, int c1, unsigned bar,
                                            unsigned long long pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar), "l"(pol)
      : "memory");
}

// Dedicated fold warps: with F = colp_folders<NP>() > 0, warps NP+1 .. NP+F fold (warp NP+1+i
// folds row i of every 4-row block) and the consumers only filter, instead of the consumers
// folding in rotation.  Measured (r02bm): NP = 7 (c5) column pass -4 % at 3 CTAs/SM (12 warps,
// 56 registers); NP = 6 (c3) +1.5 %, so the auto choice (GC_COLP_FOLDERS = -1) takes them for
// NP = 7 only; 0 / 4 force them off / on.
#ifndef GC_COLP_FOLDERS
#define GC_COLP_FOLDERS -1
#endif
#ifndef GC_COLP_FOLD_CTAS
#define GC_COLP_FOLD_CTAS 3
#endif
template <int NP>
__host__ __device__ constexpr int colp_folders() {
  return GC_COLP_STAGE_BLOCKS ? (GC_COLP_FOLDERS >= 0 ? GC_COLP_FOLDERS : (NP == 7 ? kRPS : 0)) : 0;
}
template <int NP>
__host__ __device__ constexpr int colp_ctas() { return colp_folders<NP>() ? GC_COLP_FOLD_CTAS : 3; }

template <int NP>
__global__ void __launch_bounds__(32 * (NP + 1 + colp_folders<NP>()), colp_ctas<NP>())
    k_col_o1p(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ CUtensorMap tmap4, const KParams p) {
  extern __shared__ __align__(1024) float4 smem_o1p[];
  ColPSmem<NP>& sm = *reinterpret_cast<ColPSmem<NP>*>(smem_o1p);
  constexpr int kColF = colp_folders<NP>();
  static_assert(kColF == 0 || kColF == kRPS, "fold warps: one per row of a stage block");
  constexpr unsigned BOX = NP * 32u * 8u;           // one image row: [NP pairs x 32 columns]
  constexpr unsigned DIR = kRPS * BOX;              // one direction of a stage (kRPS rows)
  constexpr unsigned SB = 2u * DIR;                 // stage: entering rows, then leaving rows
  const int nst = p.o1_stages;
  const unsigned ring = smem_u32(smem_o1p) + (unsigned)colp_head<NP>();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ncb = (p.Wd + 31) / 32;
  const int task = blockIdx.x;
  const int cb = task % ncb;
  const int sy = (task / ncb) % p.o1_nseg_y;
  const int b = task / (ncb * p.o1_nseg_y);
  const int ys = sy * p.o1_seg_y, ye = min(ys + p.o1_seg_y, p.out_rows);
  const int R = p.R;
  const int zl = 2 * R + 1;                         // steps whose leaving sample is (virtual) zero
  const int lead = (zl + kRPS - 1) / kRPS * kRPS;   // lead-in from zero state, whole stages
  const int i0 = ys - lead;                         // window centre of step 0
  const int ngroups = (lead + (ye - ys) + kRPS - 1) / kRPS;
  if (threadIdx.x == 0) {
    for (int st = 0; st < nst; st++) {
      o1_mbar_init_n(&sm.full[st], 1);
      o1_mbar_init_n(&sm.empty[st], NP);
    }
    for (int t = 0; t < kColT; t++) {
      o1_mbar_init_n(&sm.tile_full[t], NP);
      o1_mbar_init_n(&sm.tile_free[t], kColF ? kColF : NP);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  pdl_wait();                                       // planes from k_row_o1

  if (warp == NP) {                                 // ---- TMA producer (one elected lane)
    if (lane == 0) {
      unsigned long long pol_keep = 0, pol_drop = 0;
      // entering rows are read again 2W+1 steps later as leaving rows: keep them in L2
      asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_keep));
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_drop));
      const int x0 = cb * 32;
      const int ybase = b * p.in_rows;
      // kRPS rows starting at global row g0 (+1 per step) into dst
      auto load = [&](unsigned dst, int g0, unsigned bar, unsigned long long pol) {
        const int r0 = g0 - p.in_row0;
        if (g0 >= 0 && g0 + kRPS <= p.H && r0 >= 0 && r0 + kRPS <= p.in_rows) {
          GC_CHK(p, p.planes + ((long long)(ybase + r0) * NP) * p.Wd + x0, 8);                  // first and last
          GC_CHK(p, p.planes + ((long long)(ybase + r0 + kRPS) * NP - 1) * p.Wd + x0, 8);       // row of the box
          tma_2d_hint(dst, &tmap4, x0, (ybase + r0) * NP, bar, pol);            // interior: one box
        } else {
#pragma unroll 1
          for (int r = 0; r < kRPS; r++) {                                    // mirrored / clamped rows
            const int rr = min(max(mirror(g0 + r, p.H) - p.in_row0, 0), p.in_rows - 1);
            GC_CHK(p, p.planes + ((long long)(ybase + rr) * NP) * p.Wd + x0, 8);
            GC_CHK(p, p.planes + ((long long)(ybase + rr + 1) * NP - 1) * p.Wd + x0, 8);
            tma_2d_hint(dst + r * BOX, &tmap, x0, (ybase + rr) * NP, bar, pol);
          }
        }
      };
      int st = 0;
      unsigned ph = 0;
      for (int g = 0; g < ngroups; g++) {
        // (the ring is full most of the time: back off instead of spinning on the consumers'
        // issue slots)
        if (g >= nst) mbar_wait_backoff(smem_u32(&sm.empty[st]), ph ^ 1);
        const int k0 = g * kRPS;                    // first step of the group
        const bool leave = k0 + kRPS - 1 >= zl;     // some step of the group has a real leaving row
        const unsigned bar = smem_u32(&sm.full[st]);
        o1_mbar_expect_tx(&sm.full[st], leave ? SB : DIR);
        const unsigned dst = ring + st * SB;
        load(dst, p.out_row0 + i0 + k0 + R + 1, bar, pol_keep);
        if (leave) load(dst + DIR, p.out_row0 + i0 + k0 - R, bar, pol_drop);
        if (++st == nst) { st = 0; ph ^= 1; }
      }
    }
    return;
  }

  // ---- consumers: warp q = plane pair q, lane = column
  const int q = warp;
  const int x = cb * 32 + lane;
  const bool xok = x < p.Wd;
  const int xc = xok ? x : p.Wd - 1;
  float2 S0 = make_float2(0.f, 0.f), Ep = S0, Lp = S0, S[kO1K - 1], D[kO1K - 1];
#pragma unroll
  for (int t = 0; t < kO1K - 1; t++) S[t] = D[t] = make_float2(0.f, 0.f);
  // (plain C++ shared-memory accesses: ordered by the mbarrier asm's memory clobbers, free to be
  // scheduled among themselves — the loads of a stage's kRPS rows issue back to back)
  constexpr int BOXF = NP * 32, DIRF = kRPS * BOXF, SBF = 2 * DIRF;   // strides in float2
  const float2* const my_ring = reinterpret_cast<const float2*>(reinterpret_cast<const char*>(smem_o1p) +
                                                               colp_head<NP>()) + q * 32 + lane;
  float2* const my_tile = &sm.tile[0][0][q][lane];
  int st = 0;
  unsigned ph = 0;
  const float2* sbase = my_ring;                    // this lane's sample in the current stage
  // shared address of the barrier block (full[], empty[], tile_full[], tile_free[] are contiguous),
  // kept in a register: recomputed from the shared window base (S2R SR_CgaCtaId) at every use it
  // was a visible stall site of the block loop (ncu r02bc)
  unsigned bar0;
  asm volatile("mov.b32 %0, %1;" : "=r"(bar0) : "r"(smem_u32(&sm.full[0])));
  static_assert(offsetof(ColPSmem<NP>, empty) == 8 * kPDMax && offsetof(ColPSmem<NP>, tile_full) == 16 * kPDMax &&
                    offsetof(ColPSmem<NP>, tile_free) == 16 * kPDMax + 8 * kColT,
                "ColPSmem barrier block layout");
  auto advance = [&](float2 pe, float2 pl) {        // window i -> i+1
    o1_update(p, S0, S, D, f2add(pe, Lp), f2add(Ep, pl), pe, pl);
    Ep = pe;
    Lp = pl;
  };
  auto acquire = [&]() {
    mbar_wait_u32(bar0 + 8 * st, ph);
    sbase = my_ring + st * SBF;
  };
  auto release = [&]() {
    __syncwarp();
    if (lane == 0) o1_mbar_arrive_u32(bar0 + 8 * (kPDMax + st));
    if (++st == nst) { st = 0; ph ^= 1; }
  };
  // lead-in: whole stages, no output; leaving samples real from step zl on.  (The direct lead-in
  // of the row pass measured no faster here, r02al: this loop waits on the TMA ring anyway.)
  const bool filters = kColF == 0 || warp < NP;    // (fold warps skip the recursion)
#pragma unroll 1
  for (int k0 = 0; filters && k0 < lead; k0 += kRPS) {
    acquire();
#pragma unroll
    for (int r = 0; r < kRPS; r++) {
      const float2 pe = sbase[r * BOXF];
      const float2 pl = k0 + r >= zl ? sbase[DIRF + r * BOXF] : make_float2(0.f, 0.f);
      advance(pe, pl);
    }
    release();
  }
  float* const outp = p.out + b * p.out_img_stride + x;
  unsigned nguard = 0;
  const unsigned long long pol_out = l2_evict_first();
  const unsigned tf0 = bar0 + 16 * kPDMax, tr0 = tf0 + 8 * kColT;
  // Eqs. (8)-(10) for output row `row` from tile row `trow` of buffer `pbuf` (all NP pairs).
  auto fold = [&](unsigned pbuf, int trow, float* orow, float fo) {   // orow: output row, column x
    const float a = p.raw ? 0.f : centre_a(p, fo);
    const float a2 = a * a;
    float2 Q2 = make_float2(0.f, 0.f), P2 = Q2, pw2 = make_float2(1.f, a);
    float vprev = 0.f, out_raw = 0.f;
    const float2* const rt = &sm.tile[pbuf][trow][0][lane];
#pragma unroll
    for (int qq = 0; qq < NP; qq++) {
      const float2 y = rt[qq * 32];
      if (qq == 0) out_raw = y.x;
      const float2 v = f2mul(p.chat2[qq], pw2);
      Q2 = f2fma(v, y, Q2);
      P2 = f2fma(make_float2(vprev, v.x), y, P2);
      vprev = v.y;
      pw2 = f2mul(pw2, f2s(a2));
    }
    const float Q = Q2.x + Q2.y, P = P2.x + P2.y;
    if (xok) {
      float o;
      if (p.raw) {
        o = out_raw;
      } else if (Q > 0.f && isfinite(Q) && isfinite(P)) {
        o = p.t_c + p.t_h * __fdividef(P, Q);          // eq. (10) + uncentring
      } else {                                         // guard (R8)
        o = fminf(fmaxf(fo, p.L), p.U);
        nguard++;
      }
      GC_CHK(p, orow, 4);
      st_f_hint(orow, o, pol_out);
    }
  };
#if GC_COLP_STAGE_BLOCKS
  if constexpr (kColF > 0) {
    // Dedicated fold warps: consumers filter block blk into tile buffer blk % kColT (after its
    // previous block was folded), fold warp fi folds row fi of every block.
    const int nblk = (ye - ys + kRPS - 1) / kRPS;
    unsigned buf = 0, bph = 0;
    if (warp < NP) {
#pragma unroll 1
      for (int blk = 0; blk < nblk; blk++) {
        const int bs = ys + blk * kRPS;
        const int nb = min(kRPS, ye - bs);
        if (blk >= kColT) mbar_wait_u32(tr0 + 8 * buf, bph ^ 1);   // block blk - kColT folded
        float2* const tb = my_tile + buf * (kRPS * BOXF);
        acquire();
        if (nb == kRPS) {
#pragma unroll
          for (int r = 0; r < kRPS; r++) {
            const float2 pe = sbase[r * BOXF], pl = sbase[DIRF + r * BOXF];
            tb[r * BOXF] = o1_output(p, S0, S);
            advance(pe, pl);
          }
        } else {
#pragma unroll 1
          for (int r = 0; r < nb; r++) {
            const float2 pe = sbase[r * BOXF], pl = sbase[DIRF + r * BOXF];
            tb[r * BOXF] = o1_output(p, S0, S);
            advance(pe, pl);
          }
        }
        release();
        __syncwarp();
        if (lane == 0) o1_mbar_arrive_u32(tf0 + 8 * buf);
        if (++buf == kColT) {
          buf = 0;
          bph ^= 1;
        }
      }
    } else {
      const int fi = warp - NP - 1;                 // the row of every block this warp folds
      // f of the row folded kFPD blocks later, loaded now: the fold warps set the pace of the
      // pass (the consumers wait on tile_free), and one block did not cover the DRAM latency of
      // f (ncu r02fin3: the fold's first use of f was 9 % of the stall samples; r02bo: c5 column
      // pass 6.16-6.32 -> 5.88-5.97 ms at kFPD = 3)
#ifndef GC_COLP_FOLD_PREFETCH
#define GC_COLP_FOLD_PREFETCH 3
#endif
      constexpr int kFPD = GC_COLP_FOLD_PREFETCH;
      const float* const frun = row_run_ptr(p, b, p.out_row0 + ys, ye - ys);   // null if the strip spans segments
      auto frow = [&](int blk) -> float {           // f at row fi of block blk (0 past the strip)
        const int r = ys + blk * kRPS + fi;
        if (blk >= nblk || r >= ye) return 0.f;
        const float* a = frun ? frun + (long long)(r - ys) * p.Wd + xc : row_ptr(p, b, p.out_row0 + r) + xc;
        GC_CHK(p, a, 4);
        return __ldg(a);
      };
      float fq[kFPD];
#pragma unroll
      for (int k = 0; k < kFPD; k++) fq[k] = frow(k);
#pragma unroll 1
      for (int blk = 0; blk < nblk; blk++) {
        const int r = ys + blk * kRPS + fi;
        const float fo = fq[0];
#pragma unroll
        for (int k = 0; k + 1 < kFPD; k++) fq[k] = fq[k + 1];
        fq[kFPD - 1] = frow(blk + kFPD);
        // (wait even when row fi lies past the strip's end: an arrival on tile_free before block
        // blk is in could complete the buffer's previous phase while another fold warp still
        // reads it — fold warps do not filter, so nothing else keeps them within a phase)
        mbar_wait_u32(tf0 + 8 * buf, bph);          // every consumer's pair of block blk is in
        if (r < ye) fold(buf, fi, outp + (long long)r * p.Wd, fo);
        __syncwarp();
        if (lane == 0) o1_mbar_arrive_u32(tr0 + 8 * buf);
        if (++buf == kColT) {
          buf = 0;
          bph ^= 1;
        }
      }
    }
    count_guarded(p.fallback, 0xffffffffu, nguard);
    return;
  }
  // Blocks of kRPS output rows = one ring stage each (the lead-in ended on a stage boundary):
  // block blk is filtered into tile buffer blk % kColT while block blk-1 is folded from its
  // buffer; row j of block k is folded by warp (kRPS k + j) mod NP, so over NP blocks every warp
  // folds kRPS rows.  tile_full / tile_free give each warp kColT - 1 blocks of slack.
  constexpr int BR = kRPS;
  const int nrows = ye - ys;
  const int nblk = (nrows + BR - 1) / BR;
  // Row j of block k is folded by warp (kRPS k + j) mod NP, i.e. warp q folds the rows ys + q,
  // ys + q + NP, ... — tracked as a running offset and running f / output pointers instead of
  // per-block index arithmetic (the block loop's integer work was a third of its instructions).
  const float* const frun = row_run_ptr(p, b, p.out_row0 + ys, nrows);   // null if the strip spans segments
  int nr = q;                                       // offset (from ys) of the next row this warp folds
  const long long fstep = (long long)NP * p.Wd;
  const float* fpn = frun ? frun + (long long)q * p.Wd + xc : nullptr;
  float* opn = outp + (long long)(ys + q) * p.Wd;
  auto fload = [&]() -> float {
    if (fpn) {
      GC_CHK(p, fpn, 4);
      return __ldg(fpn);
    }
    GC_CHK(p, row_ptr(p, b, p.out_row0 + ys + nr) + xc, 4);
    return __ldg(row_ptr(p, b, p.out_row0 + ys + nr) + xc);
  };
  float fo = 0.f;                                   // f at the row this warp folds next
  // tile buffer of block blk / of block blk - 1 and their mbarrier phase parities (blk / kColT) & 1,
  // (blk - 1) / kColT & 1 as rolling counters (a modulo by kColT = 3 was a visible stall site)
  unsigned buf = 0, bph = 0, pbuf = 0, pph = 0;
#ifndef GC_COLP_FOLD_LAG
#define GC_COLP_FOLD_LAG 1
#endif
  // iteration blk filters block blk and folds block blk - FL: a folder may run FL - 1 blocks ahead
  // of the slowest filtering warp, a filtering warp kColT - FL blocks ahead of the slowest folder
  constexpr int FL = GC_COLP_FOLD_LAG;
  static_assert(FL >= 1 && FL < kColT, "fold lag needs kColT > FL tile buffers");
#pragma unroll 1
  for (int blk = 0; blk < nblk + FL; blk++) {
    const int pb = blk - FL;                        // block folded in this iteration
    const int pend = min(BR * (pb + 1), nrows);     // rows [0, pend) are in blocks <= pb
    const bool folds = nr < pend;                   // this warp folds a row of block pb
    if (folds) fo = fload();                        // used after the filtering
    if (blk < nblk) {                               // ---- filter block blk into tile buffer buf
      const int bs = ys + blk * BR;
      const int nb = min(BR, ye - bs);
      if (blk >= kColT) mbar_wait_u32(tr0 + 8 * buf, bph ^ 1);   // block blk - kColT folded
      float2* const tb = my_tile + buf * (BR * BOXF);
      acquire();
      if (nb == BR) {
#pragma unroll
        for (int r = 0; r < BR; r++) {
          const float2 pe = sbase[r * BOXF], pl = sbase[DIRF + r * BOXF];
          tb[r * BOXF] = o1_output(p, S0, S);       // filtered pair q at row bs + r
          advance(pe, pl);
        }
      } else {
#pragma unroll 1
        for (int r = 0; r < nb; r++) {
          const float2 pe = sbase[r * BOXF], pl = sbase[DIRF + r * BOXF];
          tb[r * BOXF] = o1_output(p, S0, S);
          advance(pe, pl);
        }
      }
      release();
      __syncwarp();
      if (lane == 0) o1_mbar_arrive_u32(tf0 + 8 * buf);
    }
    if (pb >= 0) {                                  // ---- fold this warp's rows of block pb: eqs. (8)-(10)
      if (folds) {
        mbar_wait_u32(tf0 + 8 * pbuf, pph);         // every warp's pair of block pb is in
        for (bool first = true; nr < pend; first = false) {   // (more than one row when NP < kRPS)
          if (!first) fo = fload();
          fold(pbuf, nr - BR * pb, opn, fo);
          nr += NP;
          if (fpn) fpn += fstep;
          opn += fstep;
        }
      }
      // (a warp folding nothing here frees the buffer at once: a warp reaching block pb + kColT
      // first waits for this phase, so no arrival can count towards a later one)
      __syncwarp();
      if (lane == 0) o1_mbar_arrive_u32(tr0 + 8 * pbuf);
    }
    if (pb >= 0 && ++pbuf == kColT) {
      pbuf = 0;
      pph ^= 1;
    }
    if (++buf == kColT) {
      buf = 0;
      bph ^= 1;
    }
  }
#else
  // Blocks of NP output rows: block blk is filtered into tile buffer blk % kColT while block blk-1
  // is folded (eqs. 8-10) from its buffer, warp q folding row q — every warp does the same work
  // per block.  The mbarriers tile_full / tile_free give each warp kColT - 1 blocks of slack.
  // (Ring stages hold kRPS rows, so the stage position r is a runtime counter here.)
  const int nblk = (ye - ys + NP - 1) / NP;
  int r = 0;                                        // row within the current ring stage
  float fo = 0.f;                                   // f at the row this warp folds next
#pragma unroll 1
  for (int blk = 0; blk <= nblk; blk++) {
    const int bs = ys + blk * NP;
    const int pb = blk - 1;                         // block folded in this iteration
    const int pbs = bs - NP;
    const int pnb = pb >= 0 ? min(NP, ye - pbs) : 0;
    if (pb >= 0 && q < pnb) {                       // used after the filtering
      GC_CHK(p, row_ptr(p, b, p.out_row0 + pbs + q) + xc, 4);
      fo = __ldg(row_ptr(p, b, p.out_row0 + pbs + q) + xc);
    }
    if (blk < nblk) {                               // ---- filter block blk into tile buffer blk % kColT
      const unsigned buf = blk % kColT;
      const int nb = min(NP, ye - bs);
      if (blk >= kColT) mbar_wait_u32(tr0 + 8 * buf, ((blk / kColT) - 1) & 1);   // block blk-kColT folded
      float2* const tb = my_tile + buf * (NP * BOXF);
      auto step = [&](int jj) {
        if (r == 0) acquire();
        const float2 pe = sbase[r * BOXF], pl = sbase[DIRF + r * BOXF];
        tb[jj * BOXF] = o1_output(p, S0, S);        // filtered pair q at row bs + jj
        advance(pe, pl);
        if (++r == kRPS) {
          release();
          r = 0;
        }
      };
      if (nb == NP) {
#pragma unroll
        for (int jj = 0; jj < NP; jj++) step(jj);
      } else {
#pragma unroll 1
        for (int jj = 0; jj < nb; jj++) step(jj);
      }
      __syncwarp();
      if (lane == 0) o1_mbar_arrive_u32(tf0 + 8 * buf);
    }
    if (pb >= 0) {                                  // ---- fold row q of block pb: eqs. (8)-(10)
      const unsigned pbuf = pb % kColT;
      mbar_wait_u32(tf0 + 8 * pbuf, (pb / kColT) & 1);   // every warp's pair of block pb is in
      if (q < pnb) fold(pbuf, q, outp + (long long)(pbs + q) * p.Wd, fo);
      __syncwarp();
      if (lane == 0) o1_mbar_arrive_u32(tr0 + 8 * pbuf);
    }
  }
#endif
  count_guarded(p.fallback, 0xffffffffu, nguard);
}

// ------------------------------------------------------------------ dispatch

namespace {

// TMA descriptor of the O(1) plane buffer [B*rows*NP][Wd] (8-byte elements), box 32 x NP.
bool make_o1_plane_map(CUtensorMap* map, const KParams& p, int rows_per_box = 1) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return false;
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const cuuint64_t dims[2] = {(cuuint64_t)p.Wd, (cuuint64_t)p.B * p.in_rows * p.NP};
  const cuuint64_t strides[1] = {(cuuint64_t)p.Wd * 8};
  const cuuint32_t box[2] = {32, (cuuint32_t)(p.NP * rows_per_box)};
  const cuuint32_t estr[2] = {1, 1};
  return encode(map, CU_TENSOR_MAP_DATA_TYPE_INT64, 2, (void*)p.planes, dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Resident warps of `kern` on the whole GPU (blocks of kO1Warps warps, `smem` bytes each).
template <typename K>
long long o1_resident_warps(K kern, size_t smem, int num_sms) {
  int blocks = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, kern, 32 * kO1Warps, smem) != cudaSuccess) blocks = 1;
  return (long long)std::max(1, blocks) * kO1Warps * num_sms;
}

template <int NPG, int G>
cudaError_t launch_col(const KParams& p0, cudaStream_t s) {
  constexpr int CW = 32 / G;
  CUtensorMap map;
  std::memset(&map, 0, sizeof(map));
  const bool tma = G == 1 && p0.NP <= NPG && (p0.Wd & 1) == 0 && make_o1_plane_map(&map, p0);
  auto kern = tma ? k_col_o1<NPG, G, true> : k_col_o1<NPG, G, false>;
  const size_t smem = kO1Warps * sizeof(ColO1Smem);
  static std::atomic<unsigned long long> ready[2];  // > 48 KB dynamic shared memory: opt in per device
  static std::atomic<long long> resident[2];        // (same device class for every device in a box)
  const cudaError_t e = once_per_device(ready[tma], [&]() {
    cudaError_t r = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (r == cudaSuccess) resident[tma].store(o1_resident_warps(kern, smem, p0.num_sms));
    return r;
  });
  if (e != cudaSuccess) return e;
  KParams p = p0;
  const long long ncb = (p.Wd + CW - 1) / CW;
  pick_segments(p.out_rows, ncb * p.B, 2 * p.R + 1, resident[tma].load(), 32, p.o1_seg_y, p.o1_nseg_y);
  const long long nt = ncb * p.o1_nseg_y * p.B;
  const unsigned grid = (unsigned)((nt + kO1Warps - 1) / kO1Warps);
  return launch_k(kern, dim3(grid), dim3(32 * kO1Warps), smem, s, p.ev[1] == nullptr, map, p);
}

// CTAs per SM for k_col_o1p: bounds the GPU's in-flight leaving-row windows (CTAs x 148 x
// NP x 32 x (2W+1) x 8 B) so they stay L2-resident; GC_O1P_CTAS overrides (development A/B).
int o1p_ctas_per_sm(int dflt) {
  static const int v = [] {
    const char* e = std::getenv("GC_O1P_CTAS");
    return e ? std::atoi(e) : 0;
  }();
  const int n = v > 0 ? v : dflt;
  return n < 1 ? 1 : (n > 8 ? 8 : n);
}

template <int NP>
cudaError_t launch_colp(const KParams& p0, cudaStream_t s) {
  CUtensorMap map, map4;
  std::memset(&map, 0, sizeof(map));
  std::memset(&map4, 0, sizeof(map4));
  if (!make_o1_plane_map(&map, p0) || !make_o1_plane_map(&map4, p0, kRPS)) return cudaErrorNotSupported;
  auto kern = k_col_o1p<NP>;
  constexpr int threads = 32 * (NP + 1 + colp_folders<NP>());
  // dynamic shared memory padded so that at most o1p_ctas_per_sm() CTAs fit on an SM
  int dev = 0, smem_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
  const int ctas = o1p_ctas_per_sm(colp_ctas<NP>());
  // ring depth: every stage the CTA's share of the SM's shared memory holds (a deep ring is what
  // hides the TMA latency: each step's compute is short), NP <= stages <= kPDMax
  const size_t cap = std::min<size_t>((size_t)(smem_sm > 0 ? smem_sm : 233472) / ctas - 1024, 227 * 1024);
  int nst = (int)((cap - colp_head<NP>()) / colp_stage<NP>());
  if (const char* env = std::getenv("GC_O1P_STAGES")) nst = std::min(nst, std::atoi(env));
  // (more than one fold block of rows in the ring: no starvation)
  const int min_st = (colp_block_rows<NP>() + kRPS - 1) / kRPS + (kColT > 2 ? 0 : 1);
  nst = std::max(std::max(2, min_st), std::min(nst, kPDMax));
  const size_t smem = colp_head<NP>() + (size_t)nst * colp_stage<NP>();
  static std::atomic<unsigned long long> ready{0};   // opt in to the largest ring once per device
  const cudaError_t e = once_per_device(ready, [&]() {
    return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  });
  if (e != cudaSuccess) return e;
  int blocks = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, kern, threads, smem) != cudaSuccess || blocks < 1)
    blocks = 1;
  KParams p = p0;
  p.o1_stages = nst;

  const long long ncb = (p.Wd + 31) / 32;
  {
    // y-segments: 8 per column strip (or one CTA per resident slot if that is more), none
    // shorter than twice the lead-in (r02am sweep: c3 sigma_s = 10 / 20 / 40 column pass
    // 0.442 / 0.504 / 0.528 ms with pick_segments' wave model, 0.438 / 0.463 / 0.512 at 8;
    // c5 unchanged)
    const long long base = ncb * p.B, res = (long long)blocks * p.num_sms;
    const long long lead = (2 * p.R + 1 + kRPS - 1) / kRPS * kRPS;
    long long n = std::max<long long>(8, (res + base - 1) / base);
    n = std::min<long long>(n, std::max<long long>(1, p.out_rows / (2 * lead)));
    n = std::max<long long>(1, std::min<long long>(n, p.out_rows));
    p.o1_seg_y = (int)((p.out_rows + n - 1) / n);
    p.o1_nseg_y = (p.out_rows + p.o1_seg_y - 1) / p.o1_seg_y;
  }
  static const int force_nseg = [] {                 // A/B switch (development)
    const char* v = std::getenv("GC_O1_COL_NSEG");
    return v ? std::atoi(v) : 0;
  }();
  if (force_nseg > 0) {
    p.o1_seg_y = (p.out_rows + force_nseg - 1) / force_nseg;
    p.o1_nseg_y = (p.out_rows + p.o1_seg_y - 1) / p.o1_seg_y;
  }
  const long long nt = ncb * p.o1_nseg_y * p.B;
  return launch_k(kern, dim3((unsigned)nt), dim3(threads), smem, s, p.ev[1] == nullptr, map, map4, p);
}

template <int G, int LO, int HI>
cudaError_t launch_col_g(const KParams& p, int npg, cudaStream_t s) {
  if constexpr (LO > HI) {
    return cudaErrorInvalidValue;
  } else {
    if (npg <= LO) return launch_col<LO, G>(p, s);
    return launch_col_g<G, LO + 1, HI>(p, npg, s);
  }
}

}  // namespace

cudaError_t launch_o1_two_pass(const KParams& p0, cudaStream_t s) {
  // row pass: warp tasks = 32 rows x one x-segment x one group of <= 4 plane pairs
  auto row_kern = k_row_o1;
  const size_t smem_r = (size_t)kO1Warps * sizeof(RowO1Smem);
  static std::atomic<unsigned long long> ready{0};
  static std::atomic<long long> resident_r{1};
  {
    const cudaError_t e = once_per_device(ready, [&]() {
      cudaError_t r = cudaFuncSetAttribute(row_kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_r);
      if (r == cudaSuccess) resident_r.store(o1_resident_warps(row_kern, smem_r, p0.num_sms));
      return r;
    });
    if (e != cudaSuccess) return e;
  }
  KParams p = p0;
  p.o1_groups = (p.NP + kO1RowNPG - 1) / kO1RowNPG;
  const long long nrb = (p.in_rows + 31) / 32;
  {
    // x-segments: 16 per line, or one task per resident warp if that is more (the dynamic
    // fetch balances the tasks), but segments at least twice the 2W+1 lead-in (measured: c5 and
    // c3 sigma_s = 2 / 10 best at 16, c3 sigma_s = 40 at 8 = the lead-in bound; r02ai-ak)
    const long long base = nrb * p.o1_groups * p.B, res = resident_r.load();
    long long n = std::max<long long>(16, (res + base - 1) / base);
    n = std::min<long long>(n, std::max(1, p.Wd / (2 * (2 * p.R + 1))));
    n = std::max<long long>(1, std::min<long long>(n, (p.Wd + 31) / 32));
    p.o1_seg_x = (int)(((p.Wd + n - 1) / n + 31) / 32 * 32);
    p.o1_nseg_x = (p.Wd + p.o1_seg_x - 1) / p.o1_seg_x;
  }
  static const int force_nseg = [] {                 // A/B switch (development)
    const char* v = std::getenv("GC_O1_ROW_NSEG");
    return v ? std::atoi(v) : 0;
  }();
  if (force_nseg > 0) {
    p.o1_seg_x = ((p.Wd + force_nseg - 1) / force_nseg + 31) / 32 * 32;
    p.o1_nseg_x = (p.Wd + p.o1_seg_x - 1) / p.o1_seg_x;
  }
  const long long ntr = nrb * p.o1_nseg_x * p.o1_groups * p.B;
  const long long row_ctas = std::min((ntr + kO1Warps - 1) / kO1Warps, resident_r.load() / kO1Warps);
  unsigned* const row_ctr = p.counters + 1;          // (counters[0]: the FIR column pass)
  if (p.ev[0]) cudaEventRecord(p.ev[0], s);
  cudaError_t e = cudaMemsetAsync(row_ctr, 0, sizeof(unsigned), s);
  if (e != cudaSuccess) return e;
  row_kern<<<(unsigned)std::max(1ll, row_ctas), 32 * kO1Warps, smem_r, s>>>(p, row_ctr);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (p.ev[1]) cudaEventRecord(p.ev[1], s);
  // column pass: the pair-parallel kernel (NP <= 8, even width: TMA boxes), else G lanes per
  // column with NPG = ceil(NP / G) pairs per lane
  static const bool legacy = std::getenv("GC_O1_COL_LEGACY") != nullptr;   // A/B switch (development)
  if (!legacy && p.NP <= 8 && (p.Wd & 1) == 0) {
    switch (p.NP) {
      case 1: e = launch_colp<1>(p, s); break;
      case 2: e = launch_colp<2>(p, s); break;
      case 3: e = launch_colp<3>(p, s); break;
      case 4: e = launch_colp<4>(p, s); break;
      case 5: e = launch_colp<5>(p, s); break;
      case 6: e = launch_colp<6>(p, s); break;
      case 7: e = launch_colp<7>(p, s); break;
      default: e = launch_colp<8>(p, s); break;
    }
    if (e != cudaErrorNotSupported) {
      if (p.ev[2]) cudaEventRecord(p.ev[2], s);
      return e;
    }
  }
  int G, npg;
  o1_col_split(p.NP, G, npg);
  switch (G) {
    case 1: e = launch_col_g<1, 1, 7>(p, npg, s); break;
    case 2: e = launch_col_g<2, 4, 7>(p, npg, s); break;
    case 4: e = launch_col_g<4, 4, 7>(p, npg, s); break;
    default: e = launch_col_g<8, 4, 5>(p, npg, s); break;
  }
  if (p.ev[2]) cudaEventRecord(p.ev[2], s);
  return e;
}

}  // namespace gc
