// gc_fir.cu — two-pass sm_100a pipeline for the GCF hot path.
//
//   K_row  (a1 + a2, horizontal):  one coalesced read of f per tile -> centre (eq. 17),
//          auxiliary planes F'_n = exp(-g^2/2sr^2) (g/t_h)^n for n = 0..2NP-1 (eq. 6,
//          scaled as in gc_coeffs.cpp) generated in registers, plane pair by plane
//          pair, and filtered along rows with the truncated taps of eq. (7).
//          Output: row-filtered plane pairs [NP][rows][Wd] (float2).
//   K_col  (a2 vertical + a3):  column pass of eq. (7) over each plane pair, fused with
//          the recombination of eqs. (8)-(10): P' = sum chat_n G'_n Fbar'_{n+1},
//          Q' = sum chat_n G'_n Fbar'_n, out = t_c + t_h P'/Q' (guard: DESIGN.md R8).
//
// Plane PAIRS (F'_{2p}, F'_{2p+1}) are the unit of work: every multiply-add is a packed
// FFMA2 on the pair, the tap (k_m, k_m) comes from the parameter bank.  The FIR is
// "input-stationary": each input sample is read once per thread and multiply-added into
// every output of the thread's register block that it touches, with compile-time tap
// indices (template radius W), so the FFMA count is exactly (2W+1) per output and plane.
// Radii above kMaxTemplW use the runtime-W kernels at the end of the file.
#include <cstdio>

#include "gc_device.cuh"

namespace gc {

// ------------------------------------------------------------------ K_row (templated W)

template <int W, int RX, int TXT, int TY>
__global__ void __launch_bounds__(TXT* TY) k_row_t(const KParams p) {
  constexpr int TX = TXT * RX;       // output columns per CTA
  constexpr int SW = TX + 2 * W;     // staged columns (with the horizontal halo)
  constexpr int NW = RX + 2 * W;     // inputs per thread
  extern __shared__ float4 smem_row[];
  float2* sEA = reinterpret_cast<float2*>(smem_row);   // [TY][SW] (e, e a')   = pair 0
  float2* sA2 = sEA + TY * SW;                          // [TY][SW] (a'^2, a'^2)

  const int b = blockIdx.z;
  const int x0 = blockIdx.x * TX;
  const int r0 = blockIdx.y * TY;    // relative to in_row0
  const int tid = threadIdx.y * TXT + threadIdx.x;

  // Stage f for TY rows x SW columns (coalesced along x; mirrored in x).
  for (int r = 0; r < TY; r++) {
    const int rr = r0 + r;
    if (rr >= p.in_rows) break;
    const float* src = row_ptr(p, b, p.in_row0 + rr);
    for (int c = tid; c < SW; c += TXT * TY) {
      const int gx = mirror(x0 - W + c, p.Wd);
      float a, e;
      centre(p, __ldg(src + gx), a, e);
      sEA[r * SW + c] = make_float2(e, e * a);
      sA2[r * SW + c] = make_float2(a * a, a * a);
    }
  }
  __syncthreads();

  const int r = threadIdx.y;
  const int rr = r0 + r;
  if (rr >= p.in_rows) return;
  const int xs = threadIdx.x * RX;
  float2 win[NW];
#pragma unroll
  for (int j = 0; j < NW; j++) win[j] = sEA[r * SW + xs + j];

  float2* dst = p.planes + b * p.planes_img_stride + (long long)rr * p.Wd + x0 + xs;
  const long long pstride = (long long)p.in_rows * p.Wd;
  const int nvalid = min(RX, p.Wd - (x0 + xs));

  for (int pp = 0; pp < p.NP; pp++) {
    float2 acc[RX];
#pragma unroll
    for (int i = 0; i < RX; i++) acc[i] = make_float2(0.f, 0.f);
#pragma unroll
    for (int j = 0; j < NW; j++) {
#pragma unroll
      for (int i = 0; i < RX; i++) {
        const int m = j - i;                     // tap index, output i, input j
        if (m >= 0 && m <= 2 * W) acc[i] = f2fma(p.tap2[m], win[j], acc[i]);
      }
    }
#pragma unroll
    for (int i = 0; i < RX; i++)
      if (i < nvalid) dst[i] = acc[i];
    dst += pstride;
    if (pp + 1 < p.NP) {
#pragma unroll
      for (int j = 0; j < NW; j++) win[j] = f2mul(win[j], sA2[r * SW + xs + j]);
    }
  }
}

// ------------------------------------------------------------------ K_col (templated W)

template <int W, int RY, int CY>
__global__ void __launch_bounds__(32 * CY) k_col_t(const KParams p) {
  constexpr int NW = RY + 2 * W;
  const int b = blockIdx.z;
  const int x = blockIdx.x * 32 + threadIdx.x;
  const int y0 = (blockIdx.y * CY + threadIdx.y) * RY;   // first output row, relative
  if (x >= p.Wd || y0 >= p.out_rows) return;

  // Input row j is global row g0 + j, mirrored (eq. 7 symmetric extension).  Interior
  // windows read consecutive plane-buffer rows; edge windows map each row explicitly.
  const int g0 = p.out_row0 + y0 - W;
  const int last = p.out_rows - 1;
  const bool interior = (g0 >= 0) && (g0 + NW - 1 <= p.H - 1) && (g0 - p.in_row0 >= 0) &&
                        (g0 + NW - 1 - p.in_row0 < p.in_rows) && (y0 + RY <= p.out_rows);
  const int jmax = min(RY, p.out_rows - y0) - 1 + 2 * W;   // last input row a stored output uses

  float a2[RY];
  float2 pw[RY], P2[RY], Q2[RY];
  float vpy[RY];
  float fo[RY];
#pragma unroll
  for (int i = 0; i < RY; i++) {
    const int yy = min(y0 + i, last);
    float a, e;
    fo[i] = __ldg(row_ptr(p, b, p.out_row0 + yy) + x);
    centre(p, fo[i], a, e);
    a2[i] = a * a;
    pw[i] = make_float2(1.f, a);                  // (G'_0, G'_1) = (1, a')
    P2[i] = make_float2(0.f, 0.f);
    Q2[i] = make_float2(0.f, 0.f);
    vpy[i] = 0.f;                                 // v_{-1} = 0
  }

  const float2* base = p.planes + b * p.planes_img_stride + x;
  const long long pstride = (long long)p.in_rows * p.Wd;
  for (int pp = 0; pp < p.NP; pp++) {
    float2 acc[RY];
#pragma unroll
    for (int i = 0; i < RY; i++) acc[i] = make_float2(0.f, 0.f);
    const float2* pl = base + pp * pstride;
    if (interior) {
      const float2* q = pl + (long long)(g0 - p.in_row0) * p.Wd;
#pragma unroll
      for (int j = 0; j < NW; j++) {
        const float2 v = __ldg(q + (long long)j * p.Wd);
#pragma unroll
        for (int i = 0; i < RY; i++) {
          const int m = j - i;
          if (m >= 0 && m <= 2 * W) acc[i] = f2fma(p.tap2[m], v, acc[i]);
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < NW; j++) {
        // rows feeding only outputs beyond out_rows are clamped (results not stored)
        int q = mirror(g0 + min(j, jmax), p.H) - p.in_row0;
        q = min(max(q, 0), p.in_rows - 1);
        const float2 v = __ldg(pl + (long long)q * p.Wd);
#pragma unroll
        for (int i = 0; i < RY; i++) {
          const int m = j - i;
          if (m >= 0 && m <= 2 * W) acc[i] = f2fma(p.tap2[m], v, acc[i]);
        }
      }
    }
    // eqs. (8)-(9): v_n = chat_n G'_n;  Q += v_n Fbar_n;  P += v_{n-1} Fbar_n
    const float2 c2 = p.chat2[pp];
#pragma unroll
    for (int i = 0; i < RY; i++) {
      const float2 v2 = f2mul(c2, pw[i]);
      Q2[i] = f2fma(v2, acc[i], Q2[i]);
      P2[i] = f2fma(make_float2(vpy[i], v2.x), acc[i], P2[i]);
      vpy[i] = v2.y;
      pw[i] = f2mul(pw[i], make_float2(a2[i], a2[i]));
    }
  }

  float* out = p.out + b * p.out_img_stride + x;
#pragma unroll
  for (int i = 0; i < RY; i++) {
    if (y0 + i > last) break;
    const float Q = Q2[i].x + Q2[i].y;
    const float P = P2[i].x + P2[i].y;
    float o;
    if (Q > 0.f && isfinite(Q) && isfinite(P)) {
      o = p.t_c + p.t_h * __fdividef(P, Q);       // eq. (10) + uncentring
      if (!isfinite(o)) o = p.t_c + p.t_h * (P / Q);
    } else {
      o = fminf(fmaxf(fo[i], p.L), p.U);          // guard (R8)
      if (p.fallback) atomicAdd(p.fallback, 1ull);
    }
    out[(long long)(y0 + i) * p.Wd] = o;
  }
}

// ------------------------------------------------------------------ runtime-W kernels

// Row pass for any radius: plane pairs staged in shared memory one pair at a time.
__global__ void __launch_bounds__(256) k_row_rt(const KParams p) {
  constexpr int TX = 64, TY = 4;
  extern __shared__ float4 smem_rt[];
  const int R = p.R;
  const int SW = TX + 2 * R;
  float2* sPL = reinterpret_cast<float2*>(smem_rt);   // [TY][SW] current plane pair
  float2* sA2 = sPL + TY * SW;                         // [TY][SW]
  const int b = blockIdx.z, x0 = blockIdx.x * TX, r0 = blockIdx.y * TY;
  const int tid = threadIdx.x;
  for (int r = 0; r < TY; r++) {
    const int rr = r0 + r;
    if (rr >= p.in_rows) break;
    const float* src = row_ptr(p, b, p.in_row0 + rr);
    for (int c = tid; c < SW; c += 256) {
      float a, e;
      centre(p, __ldg(src + mirror(x0 - R + c, p.Wd)), a, e);
      sPL[r * SW + c] = make_float2(e, e * a);
      sA2[r * SW + c] = make_float2(a * a, a * a);
    }
  }
  __syncthreads();
  const int r = tid / TX, xo = tid % TX;
  const int rr = r0 + r;
  const bool ok = rr < p.in_rows && x0 + xo < p.Wd;
  const long long pstride = (long long)p.in_rows * p.Wd;
  for (int pp = 0; pp < p.NP; pp++) {
    if (ok) {
      float2 acc = make_float2(0.f, 0.f);
      for (int m = 0; m <= 2 * R; m++) acc = f2fma(p.taps_g[m], sPL[r * SW + xo + m], acc);
      p.planes[b * p.planes_img_stride + pp * pstride + (long long)rr * p.Wd + x0 + xo] = acc;
    }
    __syncthreads();
    for (int idx = tid; idx < TY * SW; idx += 256) sPL[idx] = f2mul(sPL[idx], sA2[idx]);
    __syncthreads();
  }
}

// Column pass + recombination for any radius: one output pixel per thread.
__global__ void __launch_bounds__(256) k_col_rt(const KParams p) {
  const int b = blockIdx.z;
  const int x = blockIdx.x * 32 + threadIdx.x % 32;
  const int y = blockIdx.y * 8 + threadIdx.x / 32;
  if (x >= p.Wd || y >= p.out_rows) return;
  const int R = p.R;
  const int gy = p.out_row0 + y;
  float a, e;
  const float f = __ldg(row_ptr(p, b, gy) + x);
  centre(p, f, a, e);
  const float a2 = a * a;
  float2 pw = make_float2(1.f, a), P2 = make_float2(0.f, 0.f), Q2 = make_float2(0.f, 0.f);
  float vpy = 0.f;
  const long long pstride = (long long)p.in_rows * p.Wd;
  for (int pp = 0; pp < p.NP; pp++) {
    const float2* pl = p.planes + b * p.planes_img_stride + pp * pstride + x;
    float2 acc = make_float2(0.f, 0.f);
    for (int m = 0; m <= 2 * R; m++) {
      const int q = mirror(gy + m - R, p.H) - p.in_row0;
      acc = f2fma(p.taps_g[m], __ldg(pl + (long long)q * p.Wd), acc);
    }
    const float2 v2 = f2mul(p.chat2[pp], pw);
    Q2 = f2fma(v2, acc, Q2);
    P2 = f2fma(make_float2(vpy, v2.x), acc, P2);
    vpy = v2.y;
    pw = f2mul(pw, make_float2(a2, a2));
  }
  const float Q = Q2.x + Q2.y, P = P2.x + P2.y;
  float o;
  if (Q > 0.f && isfinite(Q) && isfinite(P)) {
    o = p.t_c + p.t_h * (P / Q);
  } else {
    o = fminf(fmaxf(f, p.L), p.U);
    if (p.fallback) atomicAdd(p.fallback, 1ull);
  }
  p.out[b * p.out_img_stride + (long long)y * p.Wd + x] = o;
}

// ------------------------------------------------------------------ dispatch

namespace {

template <int W>
cudaError_t launch_t(const KParams& p, cudaStream_t s) {
  constexpr int RX = (W <= 16) ? 16 : 8;
  constexpr int TXT = 8, TY = 16;
  constexpr int RY = 8, CY = 8;
  constexpr int TX = TXT * RX;
  const size_t smem = (size_t)TY * (TX + 2 * W) * 16;
  auto kr = k_row_t<W, RX, TXT, TY>;
  cudaError_t e = cudaFuncSetAttribute(kr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 gr((p.Wd + TX - 1) / TX, (p.in_rows + TY - 1) / TY, p.B);
  if (p.ev[0]) cudaEventRecord(p.ev[0], s);
  kr<<<gr, dim3(TXT, TY), smem, s>>>(p);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (p.ev[1]) cudaEventRecord(p.ev[1], s);
  dim3 gc((p.Wd + 31) / 32, (p.out_rows + RY * CY - 1) / (RY * CY), p.B);
  k_col_t<W, RY, CY><<<gc, dim3(32, CY), 0, s>>>(p);
  e = cudaGetLastError();
  if (p.ev[2]) cudaEventRecord(p.ev[2], s);
  return e;
}

template <int W>
struct Table {
  static cudaError_t go(const KParams& p, cudaStream_t s) {
    if (p.R == W) return launch_t<W>(p, s);
    return Table<W - 1>::go(p, s);
  }
};
template <>
struct Table<0> {
  static cudaError_t go(const KParams&, cudaStream_t) { return cudaErrorInvalidValue; }
};

cudaError_t launch_rt(const KParams& p, cudaStream_t s) {
  const size_t smem = (size_t)4 * (64 + 2 * p.R) * 16;
  cudaError_t e = cudaFuncSetAttribute(k_row_rt, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 gr((p.Wd + 63) / 64, (p.in_rows + 3) / 4, p.B);
  if (p.ev[0]) cudaEventRecord(p.ev[0], s);
  k_row_rt<<<gr, 256, smem, s>>>(p);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (p.ev[1]) cudaEventRecord(p.ev[1], s);
  dim3 gc((p.Wd + 31) / 32, (p.out_rows + 7) / 8, p.B);
  k_col_rt<<<gc, 256, 0, s>>>(p);
  e = cudaGetLastError();
  if (p.ev[2]) cudaEventRecord(p.ev[2], s);
  return e;
}

}  // namespace

cudaError_t launch_fir_two_pass(const KParams& p, cudaStream_t stream) {
  if (p.R >= 1 && p.R <= kMaxTemplW) return Table<kMaxTemplW>::go(p, stream);
  return launch_rt(p, stream);
}

}  // namespace gc
