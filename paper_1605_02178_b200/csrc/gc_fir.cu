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
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstring>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "gc_device.cuh"

namespace gc {

// ------------------------------------------------------------------ K_row (templated W)
//
// Persistent grid; the unit of work is a WARP task: 4 image rows x 128 columns.
// Lane = (row r = lane/8, column block tx = lane%8); each lane owns RX = 16 consecutive
// outputs.  The warp stages its 4 rows of f (+ horizontal halo) in a warp-private,
// bank-conflict-free shared-memory slice holding the CURRENT plane pair
// (F'_{2p}, F'_{2p+1}) and a'^2; between pairs every element is advanced once
// (psi <- psi a'^2, FMUL2).  The FIR streams the lane's RX + 2W inputs from shared
// memory input-stationary (each input multiply-added into every output it touches, with
// compile-time tap indices), and each filtered pair is written as full rows with
// 16-byte stores after a shared-memory transpose-free staging.

constexpr int kRowWarpsPerCta = 1;

template <int W>
struct RowCfg {
  static constexpr int RX = 16;
  static constexpr int WCOLS = 8 * RX;          // output columns per warp task
  static constexpr int SW = WCOLS + 2 * W;      // staged columns
  static constexpr int NW = RX + 2 * W;         // inputs per lane
  static constexpr int NLD = (SW + 31) / 32;    // staged elements per lane per row
  // +1 pair every 16: the 8 lanes of a row (stride 16 columns) hit distinct bank pairs
  static __device__ __forceinline__ int pad(int c) { return c + (c >> 4); }
  static constexpr int SWP0 = SW + (SW >> 4) + 1;
  static constexpr int SWP = SWP0 + (24 - SWP0 % 16) % 16;   // row stride = 8 (mod 16) pairs
  static constexpr int OWP0 = WCOLS + (WCOLS >> 4) + 1;
  static constexpr int OWP = OWP0 + (24 - OWP0 % 16) % 16;
  static constexpr int A2W = SW + 1;                         // scalar a'^2 row stride
  static constexpr int SMEM_WARP = (4 * SWP + 4 * OWP) * 8 + 4 * A2W * 4;
};

template <int W>
__global__ void __launch_bounds__(32 * kRowWarpsPerCta, 16) k_row_t(const KParams p, unsigned* col_task_ctr) {
  if (blockIdx.x == 0 && threadIdx.x == 0) *col_task_ctr = 0u;   // consumed by k_col_t (stream-ordered)
  pdl_trigger();
  using C = RowCfg<W>;
  constexpr int RX = C::RX;
  extern __shared__ float4 smem_row[];
  const int lane = threadIdx.x & 31;
  float2* sPsi = reinterpret_cast<float2*>(smem_row);        // [4][SWP] current plane pair
  float2* sO = sPsi + 4 * C::SWP;                              // [4][OWP]
  float* sA2 = reinterpret_cast<float*>(sO + 4 * C::OWP);      // [4][A2W] a'^2

  const int ncb = (p.Wd + C::WCOLS - 1) / C::WCOLS;
  const int nrb = (p.in_rows + 3) / 4;
  const int r = lane >> 3, tx = lane & 7;
  const long long pstride = (long long)p.in_rows * p.Wd;
  const bool vec = (p.Wd & 1) == 0;

  const int task = blockIdx.x;
  const int cb = task % ncb;
  const int rb = (task / ncb) % nrb;
  const int b = task / (ncb * nrb);
  const int x0 = cb * C::WCOLS, y0 = rb * 4;
  const bool xint = (x0 - W >= 0) && (x0 + C::WCOLS + W <= p.Wd);

  // 1. stage f: 4 rows x SW columns (mirrored in x at the image edges), loads first
  float fv[4][C::NLD];
#pragma unroll
  for (int rr = 0; rr < 4; rr++) {
    const float* src = row_ptr(p, b, p.in_row0 + min(y0 + rr, p.in_rows - 1));
#pragma unroll
    for (int k = 0; k < C::NLD; k++) {
      const int c = lane + 32 * k;
      const int gx = xint ? x0 - W + c : mirror(x0 - W + c, p.Wd);
      if (c < C::SW) GC_CHK(p, src + gx, 4);
      fv[rr][k] = (c < C::SW) ? __ldg(src + gx) : 0.f;
    }
  }
#pragma unroll
  for (int rr = 0; rr < 4; rr++) {
#pragma unroll
    for (int k = 0; k < C::NLD; k++) {
      const int c = lane + 32 * k;
      if (c < C::SW) {
        float a, e;
        centre(p, fv[rr][k], a, e);
        if (p.raw) { e = fv[rr][k]; a = 0.f; }                      // gc_gaussian: (f, 0)
        sPsi[rr * C::SWP + C::pad(c)] = make_float2(e, e * a);      // pair 0: e (1, a')
        sA2[rr * C::A2W + c] = a * a;
      }
    }
  }
  __syncwarp();

  const float2* wrow = sPsi + r * C::SWP;
  float2* drow = p.planes + b * p.planes_img_stride + (long long)y0 * p.Wd + x0;
  for (int pp = 0; pp < p.NP; pp++) {
    float2 acc[RX];
#pragma unroll
    for (int i = 0; i < RX; i++) acc[i] = make_float2(0.f, 0.f);
#pragma unroll
    for (int j = 0; j < C::NW; j++) {
      const float2 v = wrow[C::pad(RX * tx + j)];
#pragma unroll
      for (int i = 0; i < RX; i++) {
        const int m = j - i;
        if (m >= 0 && m <= 2 * W) acc[i] = f2fma(make_float2(p.tap[m], p.tap[m]), v, acc[i]);
      }
    }
    // 2. stage the pair, then 4 rows of 128 pairs with 16-byte stores
#pragma unroll
    for (int i = 0; i < RX; i++) sO[r * C::OWP + C::pad(RX * tx + i)] = acc[i];
    __syncwarp();
#pragma unroll
    for (int rr = 0; rr < 4; rr++) {
      if (y0 + rr < p.in_rows) {
        float2* d = drow + pp * pstride + (long long)rr * p.Wd;
#pragma unroll
        for (int h = 0; h < 2; h++) {
          const int c = 2 * lane + 64 * h;
          const float2 u = sO[rr * C::OWP + C::pad(c)], v = sO[rr * C::OWP + C::pad(c + 1)];
          if (vec && x0 + c + 1 < p.Wd) {
            GC_CHK(p, d + c, 16);
            *reinterpret_cast<float4*>(d + c) = make_float4(u.x, u.y, v.x, v.y);
          } else {
            if (x0 + c < p.Wd) { GC_CHK(p, d + c, 8); d[c] = u; }
            if (x0 + c + 1 < p.Wd) { GC_CHK(p, d + c + 1, 8); d[c + 1] = v; }
          }
        }
      }
    }
    // 3. next plane pair: psi <- psi a'^2, once per staged element (loads, then stores)
    if (pp + 1 < p.NP) {
      float2 u[4][C::NLD];
      float w[4][C::NLD];
#pragma unroll
      for (int rr = 0; rr < 4; rr++)
#pragma unroll
        for (int k = 0; k < C::NLD; k++) {
          const int c = min(lane + 32 * k, C::SW - 1);
          u[rr][k] = sPsi[rr * C::SWP + C::pad(c)];
          w[rr][k] = sA2[rr * C::A2W + c];
        }
#pragma unroll
      for (int rr = 0; rr < 4; rr++)
#pragma unroll
        for (int k = 0; k < C::NLD; k++) {
          const int c = lane + 32 * k;
          if (c < C::SW) sPsi[rr * C::SWP + C::pad(c)] = f2mul(u[rr][k], make_float2(w[rr][k], w[rr][k]));
        }
    }
    __syncwarp();
  }
}

// ------------------------------------------------------------------ K_col (templated W)
//
// Persistent, warp-specialised pipeline.  CTA = 1 producer warp + 4 consumer warps.
// Task: 32 image columns x 32 output rows; consumer warp c owns rows [8c, 8c+8) of the
// task, lane = column.  A "stage" is one plane pair of one task: the (32 + 2W)-row x
// 32-column strip of the row-pass buffer that the task's column FIR reads.  The producer
// fills a 4-deep ring of stage buffers: one TMA 2-D tensor copy per stage for interior
// strips (cp.async.bulk.tensor, OOB columns zero-filled), one bulk copy per row for strips
// that need the symmetric extension at the top/bottom edge, and plain loads for odd
// widths.  full[s] / empty[s] mbarriers hand buffers between producer and consumers, so
// consumer warps never meet at a CTA barrier.  Consumers run the FIR input-stationary
// from shared memory (exact tap count) and fold each filtered pair into P and Q
// (eqs. 8-9) in registers; eq. (10) and the guard are applied at the end of the task.

constexpr int kColConsumers = 4;
constexpr int kColStages = 3;

template <int W>
struct ColCfg {
  static constexpr int RY = 8;
  static constexpr int TROWS = kColConsumers * RY;     // output rows per task
  static constexpr int NJ = TROWS + 2 * W;             // strip rows per stage
  static constexpr int NW = RY + 2 * W;
  static constexpr int BUF = NJ * 32;                  // float2 per stage buffer
  static constexpr int BUFB = BUF * 8;
  static constexpr int SMEM = kColStages * BUFB + 2 * kColStages * 8 + kColStages * 4 + 128;
};

__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(s) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
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
__device__ __forceinline__ void bulk_g2s(void* smem, const void* gmem, unsigned bytes, unsigned long long* bar) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(s),
               "l"(gmem), "r"(bytes), "r"(b)
               : "memory");
}
__device__ __forceinline__ void tma_2d(void* smem, const CUtensorMap* map, int c0, int c1, unsigned long long* bar) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(s),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(b)
      : "memory");
}

template <int W>
__global__ void __launch_bounds__(32 * (kColConsumers + 1), 4)
    k_col_t(const __grid_constant__ CUtensorMap tmap, const KParams p, unsigned* task_ctr) {
  using C = ColCfg<W>;
  constexpr int RY = C::RY;
  // dynamic shared memory starts at offset 0 of the CTA's window (no static smem here), so it
  // is 1024-byte aligned; no integer arithmetic on the pointer, so every access stays LDS/STS
  extern __shared__ __align__(1024) float4 smem_col[];
  char* base = reinterpret_cast<char*>(smem_col);
  float2* sB = reinterpret_cast<float2*>(base);                                         // [S][NJ][32]
  unsigned long long* full = reinterpret_cast<unsigned long long*>(base + kColStages * C::BUFB);
  unsigned long long* empty = full + kColStages;
  int* stage_task = reinterpret_cast<int*>(empty + kColStages);                        // [S]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  const int ncb = (p.Wd + 31) / 32;
  const int nrb = (p.out_rows + C::TROWS - 1) / C::TROWS;
  const int ntask = ncb * nrb * p.B;
  const long long pstride = (long long)p.in_rows * p.Wd;
  const int last = p.out_rows - 1;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kColStages; i++) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kColConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  pdl_wait();                                     // planes and task counter from k_row_t

  if (warp == kColConsumers) {
    // ------------------------------------------------ producer warp: fetch tasks dynamically,
    // fill stage buffers (one stage = one plane pair of one task), tag each with its task
    const bool tma_ok = (p.Wd & 1) == 0;          // 16-byte global row stride
    int k = 0;
    for (;;) {
      int task = 0;
      if (lane == 0) task = (int)atomicAdd(task_ctr, 1u);
      task = __shfl_sync(0xffffffffu, task, 0);
      const bool done = task >= ntask;
      const int rb = task % nrb;
      const int cb = (task / nrb) % ncb;
      const int b = task / (nrb * ncb);
      const int x0 = cb * 32, y0 = rb * C::TROWS;
      const int g0 = p.out_row0 + y0 - W;
      const int jmax = min(C::TROWS, p.out_rows - y0) - 1 + 2 * W;
      const bool interior = (g0 >= 0) && (g0 + C::NJ - 1 <= p.H - 1) && (g0 - p.in_row0 >= 0) &&
                            (g0 + C::NJ - 1 - p.in_row0 < p.in_rows) && (jmax == C::NJ - 1);
      const int npairs = done ? 1 : p.NP;
      for (int pp = 0; pp < npairs; pp++, k++) {
        const int s = k % kColStages;
        if (k >= kColStages) mbar_wait(&empty[s], ((k / kColStages) - 1) & 1);
        if (lane == 0) stage_task[s] = done ? -1 : task;
        float2* dst = sB + s * C::BUF;
        if (done) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&full[s]);   // sentinel: no more tasks
        } else if (tma_ok && interior) {
          if (lane == 0) {
            GC_CHK(p, p.planes + ((long long)(b * p.NP + pp) * p.in_rows + (g0 - p.in_row0)) * p.Wd + x0, 8);
            GC_CHK(p, p.planes + ((long long)(b * p.NP + pp) * p.in_rows + (g0 - p.in_row0) + C::NJ - 1) * p.Wd + x0, 8);
            mbar_expect_tx(&full[s], C::BUFB);
            tma_2d(dst, &tmap, x0, (b * p.NP + pp) * p.in_rows + (g0 - p.in_row0), &full[s]);
          }
        } else if (tma_ok && x0 + 32 <= p.Wd) {
          // symmetric extension at the top / bottom: one bulk copy per strip row
          if (lane == 0) mbar_expect_tx(&full[s], C::BUFB);
          __syncwarp();
          const float2* pl = p.planes + b * p.planes_img_stride + pp * pstride + x0;
          for (int j = lane; j < C::NJ; j += 32) {
            int q = mirror(g0 + min(j, jmax), p.H) - p.in_row0;
            q = min(max(q, 0), p.in_rows - 1);
            GC_CHK(p, pl + (long long)q * p.Wd, 256);
            bulk_g2s(dst + j * 32, pl + (long long)q * p.Wd, 256, &full[s]);
          }
        } else {
          // odd width or right-edge strip at an edge row: plain loads
          const float2* pl = p.planes + b * p.planes_img_stride + pp * pstride + x0;
          for (int j = 0; j < C::NJ; j++) {
            int q = mirror(g0 + min(j, jmax), p.H) - p.in_row0;
            q = min(max(q, 0), p.in_rows - 1);
            if (x0 + lane < p.Wd) GC_CHK(p, pl + (long long)q * p.Wd + lane, 8);
            dst[j * 32 + lane] = (x0 + lane < p.Wd) ? pl[(long long)q * p.Wd + lane] : make_float2(0.f, 0.f);
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&full[s]);
        }
      }
      if (done) break;
    }
    return;
  }

  // ------------------------------------------------ consumer warps
  const int seg = warp;
  unsigned nguard = 0;                             // guarded outputs of this lane (R8)
  float fo[RY], av[RY], P[RY], Q[RY], vpy[RY], pwx[RY], raw0[RY];
  int b = 0, x = 0, y0 = 0;
  int pp = 0;                                      // stages arrive in (task, pair) order
  for (int k = 0;; k++, pp = (pp + 1 == p.NP) ? 0 : pp + 1) {
    const int s = k % kColStages;
    mbar_wait(&full[s], (k / kColStages) & 1);
    const int task = stage_task[s];
    if (task < 0) break;
    if (pp == 0) {
      const int rb = task % nrb;
      const int cb = (task / nrb) % ncb;
      b = task / (nrb * ncb);
      y0 = rb * C::TROWS;
      x = cb * 32 + lane;
      // issue the loads of f now, use them after this pair's FIR (latency overlapped)
      const int ya = y0 + RY * seg;
      const float* run = ya + RY - 1 <= last ? row_run_ptr(p, b, p.out_row0 + ya, RY) : nullptr;
      if (run) {
#pragma unroll
        for (int i = 0; i < RY; i++) {
          if (x < p.Wd) GC_CHK(p, run + (long long)i * p.Wd + x, 4);
          fo[i] = (x < p.Wd) ? __ldg(run + (long long)i * p.Wd + x) : 0.f;
        }
      } else {
#pragma unroll
        for (int i = 0; i < RY; i++) {
          const int yy = min(ya + i, last);
          if (x < p.Wd) GC_CHK(p, row_ptr(p, b, p.out_row0 + yy) + x, 4);
          fo[i] = (x < p.Wd) ? __ldg(row_ptr(p, b, p.out_row0 + yy) + x) : 0.f;
        }
      }
    }
    const float2* col = sB + s * C::BUF + (RY * seg) * 32 + lane;
    float2 acc[RY];
#pragma unroll
    for (int i = 0; i < RY; i++) acc[i] = make_float2(0.f, 0.f);
#pragma unroll
    for (int j = 0; j < C::NW; j++) {
      const float2 v = col[j * 32];
#pragma unroll
      for (int i = 0; i < RY; i++) {
        const int m = j - i;
        if (m >= 0 && m <= 2 * W) acc[i] = f2fma(make_float2(p.tap[m], p.tap[m]), v, acc[i]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);       // strip no longer needed by this warp
    if (pp == 0) {
#pragma unroll
      for (int i = 0; i < RY; i++) {
        raw0[i] = acc[i].x;
        float a, e;
        centre(p, fo[i], a, e);
        av[i] = a;
        pwx[i] = 1.f;          // G'_{2p} = a'^{2p}
        P[i] = 0.f;
        Q[i] = 0.f;
        vpy[i] = 0.f;          // v_{-1} = 0
      }
    }
    // eqs. (8)-(9) with v_n = chat_n G'_n:  Q += v_n Fbar_n,  P += v_{n-1} Fbar_n
    const float2 c2 = p.chat2[pp];
#pragma unroll
    for (int i = 0; i < RY; i++) {
      const float v0 = c2.x * pwx[i];
      const float v1 = c2.y * (pwx[i] * av[i]);
      Q[i] = fmaf(v0, acc[i].x, Q[i]);
      Q[i] = fmaf(v1, acc[i].y, Q[i]);
      P[i] = fmaf(vpy[i], acc[i].x, P[i]);
      P[i] = fmaf(v0, acc[i].y, P[i]);
      vpy[i] = v1;
      pwx[i] *= av[i] * av[i];
    }
    if (pp == p.NP - 1 && x < p.Wd) {
      float* out = p.out + b * p.out_img_stride + x;
#pragma unroll
      for (int i = 0; i < RY; i++) {
        const int yy = y0 + RY * seg + i;
        if (yy > last) break;
        const float Qi = Q[i], Pi = P[i];
        float o;
        if (p.raw) {
          o = raw0[i];
        } else if (Qi > 0.f && isfinite(Qi) && isfinite(Pi)) {
          o = p.t_c + p.t_h * __fdividef(Pi, Qi);        // eq. (10) + uncentring
        } else {                                          // guard (R8)
          o = fminf(fmaxf(fo[i], p.L), p.U);
          nguard++;
        }
        GC_CHK(p, &out[(long long)yy * p.Wd], 4);
        out[(long long)yy * p.Wd] = o;
      }
    }
  }
  count_guarded(p.fallback, 0xffffffffu, nguard);
}

// ------------------------------------------------------------------ runtime-W kernels

// Row pass for any radius: plane pairs staged in shared memory one pair at a time.
__global__ void __launch_bounds__(256) k_row_rt(const KParams p) {
  pdl_trigger();
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
      GC_CHK(p, src + mirror(x0 - R + c, p.Wd), 4);
      const float fv = __ldg(src + mirror(x0 - R + c, p.Wd));
      centre(p, fv, a, e);
      if (p.raw) { e = fv; a = 0.f; }
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
      GC_CHK(p, &p.planes[b * p.planes_img_stride + pp * pstride + (long long)rr * p.Wd + x0 + xo], 8);
      p.planes[b * p.planes_img_stride + pp * pstride + (long long)rr * p.Wd + x0 + xo] = acc;
    }
    __syncthreads();
    for (int idx = tid; idx < TY * SW; idx += 256) sPL[idx] = f2mul(sPL[idx], sA2[idx]);
    __syncthreads();
  }
}

// Column pass + recombination for any radius: one output pixel per thread.
__global__ void __launch_bounds__(256) k_col_rt(const KParams p) {
  pdl_wait();
  const int b = blockIdx.z;
  const int x = blockIdx.x * 32 + threadIdx.x % 32;
  const int y = blockIdx.y * 8 + threadIdx.x / 32;
  if (x >= p.Wd || y >= p.out_rows) return;
  const int R = p.R;
  const int gy = p.out_row0 + y;
  float a, e;
  GC_CHK(p, row_ptr(p, b, gy) + x, 4);
  const float f = __ldg(row_ptr(p, b, gy) + x);
  centre(p, f, a, e);
  const float a2 = a * a;
  float2 pw = make_float2(1.f, a), P2 = make_float2(0.f, 0.f), Q2 = make_float2(0.f, 0.f);
  float vpy = 0.f, raw0 = 0.f;
  const long long pstride = (long long)p.in_rows * p.Wd;
  for (int pp = 0; pp < p.NP; pp++) {
    const float2* pl = p.planes + b * p.planes_img_stride + pp * pstride + x;
    float2 acc = make_float2(0.f, 0.f);
    for (int m = 0; m <= 2 * R; m++) {
      const int q = mirror(gy + m - R, p.H) - p.in_row0;
      GC_CHK(p, pl + (long long)q * p.Wd, 8);
      acc = f2fma(p.taps_g[m], __ldg(pl + (long long)q * p.Wd), acc);
    }
    if (pp == 0) raw0 = acc.x;
    const float2 v2 = f2mul(p.chat2[pp], pw);
    Q2 = f2fma(v2, acc, Q2);
    P2 = f2fma(make_float2(vpy, v2.x), acc, P2);
    vpy = v2.y;
    pw = f2mul(pw, make_float2(a2, a2));
  }
  const float Q = Q2.x + Q2.y, P = P2.x + P2.y;
  float o;
  unsigned guarded = 0;
  if (p.raw) {
    o = raw0;
  } else if (Q > 0.f && isfinite(Q) && isfinite(P)) {
    o = p.t_c + p.t_h * (P / Q);
  } else {
    o = fminf(fmaxf(f, p.L), p.U);
    guarded = 1;
  }
  count_guarded(p.fallback, __activemask(), guarded);
  GC_CHK(p, &p.out[b * p.out_img_stride + (long long)y * p.Wd + x], 4);
  p.out[b * p.out_img_stride + (long long)y * p.Wd + x] = o;
}

// ------------------------------------------------------------------ dispatch

namespace {

// TMA descriptor of the row-pass buffer seen as a 2-D tensor of 8-byte elements:
// [B * NP * in_rows rows][Wd columns], box = 32 columns x `box_rows` rows.
bool make_plane_map(CUtensorMap* map, const KParams& p, int box_rows) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return false;
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  if ((p.Wd & 1) != 0) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)p.Wd, (cuuint64_t)p.B * p.NP * p.in_rows};
  const cuuint64_t strides[1] = {(cuuint64_t)p.Wd * 8};
  const cuuint32_t box[2] = {32, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  return encode(map, CU_TENSOR_MAP_DATA_TYPE_INT64, 2, (void*)p.planes, dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int W>
cudaError_t launch_t(const KParams& p, cudaStream_t s) {
  using CR = RowCfg<W>;
  using CC = ColCfg<W>;
  const size_t smem_r = (size_t)kRowWarpsPerCta * CR::SMEM_WARP;
  const size_t smem_c = (size_t)CC::SMEM;
  auto kr = k_row_t<W>;
  auto kc = k_col_t<W>;
  static std::atomic<unsigned long long> ready{0};   // per instantiation and device
  static std::atomic<int> occ_c_s{1};
  cudaError_t e0 = once_per_device(ready, [&]() {
    cudaError_t e = cudaFuncSetAttribute(kr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_r);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(kc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_c);
    int oc = 0;
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&oc, kc, 32 * (kColConsumers + 1), smem_c);
    if (e == cudaSuccess) occ_c_s.store(std::max(oc, 1));
    return e;
  });
  if (e0 != cudaSuccess) return e0;
  const int occ_c = occ_c_s.load();
  CUtensorMap map;
  std::memset(&map, 0, sizeof(map));
  if ((p.Wd & 1) == 0 && !make_plane_map(&map, p, CC::NJ)) return cudaErrorInvalidValue;
  const long long ntr = (long long)((p.Wd + CR::WCOLS - 1) / CR::WCOLS) * ((p.in_rows + 3) / 4) * p.B;
  const long long gr = ntr;                // one warp task per CTA
  const long long ntc = (long long)((p.Wd + 31) / 32) * ((p.out_rows + CC::TROWS - 1) / CC::TROWS) * p.B;
  const long long gc = std::min<long long>(ntc, (long long)occ_c * p.num_sms);   // persistent, dynamic tasks
  if (p.ev[0]) cudaEventRecord(p.ev[0], s);
  kr<<<(unsigned)gr, 32 * kRowWarpsPerCta, smem_r, s>>>(p, p.counters);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (p.ev[1]) cudaEventRecord(p.ev[1], s);
  e = launch_k(kc, dim3((unsigned)gc), dim3(32 * (kColConsumers + 1)), smem_c, s, p.ev[1] == nullptr, map, p,
               p.counters);
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
  static std::atomic<unsigned long long> ready{0};
  cudaError_t e = once_per_device(ready, [&]() {   // the largest radius's size: covers every call
    return cudaFuncSetAttribute(k_row_rt, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)((size_t)4 * (64 + 2 * kMaxFirW) * 16));
  });
  if (e != cudaSuccess) return e;
  dim3 gr((p.Wd + 63) / 64, (p.in_rows + 3) / 4, p.B);
  if (p.ev[0]) cudaEventRecord(p.ev[0], s);
  k_row_rt<<<gr, 256, smem, s>>>(p);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (p.ev[1]) cudaEventRecord(p.ev[1], s);
  dim3 gc((p.Wd + 31) / 32, (p.out_rows + 7) / 8, p.B);
  e = launch_k(k_col_rt, gc, dim3(256), 0, s, p.ev[1] == nullptr, p);
  if (p.ev[2]) cudaEventRecord(p.ev[2], s);
  return e;
}

}  // namespace

cudaError_t launch_fir_two_pass(const KParams& p, cudaStream_t stream) {
  if (fused_fir_applies(p)) return launch_fused_fir(p, stream);
  if (p.R >= 1 && p.R <= kMaxTemplW) return Table<kMaxTemplW>::go(p, stream);
  return launch_rt(p, stream);
}

}  // namespace gc
