// gc_fused.cu — small-image FIR path: steps a1-a3 of the GCF (eq. 7 with the planes of
// eqs. 5-6, recombination and division of eqs. 8-10) for one output tile per CTA, both passes of
// eq. (7) in shared memory.
//
// The two-pass FIR path (gc_fir.cu) writes the N+2 planes to global memory between its passes and
// costs two launches with a pipeline fill and drain each; on a 256^2 or 1024^2 image that fixed
// cost is most of the call (profiles/r01_ab_experiments.md: t(B) = 26 us + 30 us B at c2).  Here
// a CTA owns a 32-column x TY-row output tile: it stages the (TY + 2W) x (32 + 2W) input region
// once (mirrored as in the two-pass path), keeps the current plane pair of the region in shared
// memory, and per pair runs the row FIR over the region rows, the column FIR over the tile and the
// eq. (8)-(9) accumulation in registers.  The halo columns are filtered by every tile that needs
// them (a (32 + 2W) / 32 row-pass overhead), in exchange for no plane round trip and one launch.
//
// Arithmetic is the two-pass path's, operation by operation (the same staging (e, e a'), the same
// psi <- psi a'^2 update, taps summed in ascending m, the same recombination order), so the two
// paths agree bit for bit (tests/test_gpu_fused.py).
#include <algorithm>
#include <atomic>
#include <cstdlib>

#include "gc_device.cuh"

namespace gc {
namespace {

constexpr int kFuTX = 32;         // tile columns
constexpr int kFuThreads = 256;   // 8 warps

template <int W, int TY>
struct FuCfg {
  static constexpr int RW = kFuTX + 2 * W;                  // region columns
  static constexpr int RH = TY + 2 * W;                     // region rows
  static constexpr int RY = TY / (kFuThreads / kFuTX);      // column pass: output rows per thread
  // row pass: consecutive outputs per item, 4 when 8 would leave threads idle (short tiles)
  static constexpr int RX = RH * (kFuTX / 8) >= 3 * kFuThreads / 4 ? 8 : 4;
  static constexpr int NF = RH * RW;
  static constexpr size_t OFF_A2 = (size_t)NF * sizeof(float2);
  static constexpr size_t OFF_R = (OFF_A2 + (size_t)NF * sizeof(float) + 15) / 16 * 16;
  static constexpr size_t SMEM = OFF_R + (size_t)RH * kFuTX * sizeof(float2);
};

template <int W, int TY>
__global__ void __launch_bounds__(kFuThreads) k_fused_fir(const KParams p) {
  using C = FuCfg<W, TY>;
  extern __shared__ float4 smem_fu[];
  float2* const sF = reinterpret_cast<float2*>(smem_fu);                                  // [RH][RW] pair
  float* const sA2 = reinterpret_cast<float*>(reinterpret_cast<char*>(smem_fu) + C::OFF_A2);  // [RH][RW] a'^2
  float2* const sR = reinterpret_cast<float2*>(reinterpret_cast<char*>(smem_fu) + C::OFF_R);  // [RH][32] row-filtered
  const int ntx = (p.Wd + kFuTX - 1) / kFuTX, nty = (p.out_rows + TY - 1) / TY;
  const int t = blockIdx.x;
  const int tx0 = (t % ntx) * kFuTX;
  const int ty0 = ((t / ntx) % nty) * TY;
  const int b = t / (ntx * nty);

  // column-pass ownership: column x of the tile, rows i0 .. i0 + RY - 1; f at those outputs is
  // loaded first (its latency overlaps the region staging)
  const int cx = threadIdx.x % kFuTX, i0 = (threadIdx.x / kFuTX) * C::RY;
  const int x = tx0 + cx;
  float fo[C::RY], av[C::RY], P[C::RY], Q[C::RY], vpy[C::RY], pwx[C::RY], raw0[C::RY];
#pragma unroll
  for (int i = 0; i < C::RY; i++) {
    const int yy = min(ty0 + i0 + i, p.out_rows - 1);
    if (x < p.Wd) GC_CHK(p, row_ptr(p, b, p.out_row0 + yy) + x, 4);
    fo[i] = x < p.Wd ? __ldg(row_ptr(p, b, p.out_row0 + yy) + x) : 0.f;
  }

  // 1. the input region, mirrored at the image edges and mapped to the window's rows as
  //    the two-pass path does: pair 0 = e (1, a'), and a'^2 for the pair update.  Loads in batches
  //    of kFuSB independent ones per thread, then the centring.
  constexpr int kFuSB = 8;
  for (int k0 = threadIdx.x; k0 < C::NF; k0 += kFuThreads * kFuSB) {
    float fv[kFuSB];
#pragma unroll
    for (int u = 0; u < kFuSB; u++) {
      const int k = k0 + u * kFuThreads;
      fv[u] = 0.f;
      if (k < C::NF) {
        const int i = k / C::RW, c = k - i * C::RW;
        const int g = p.out_row0 + ty0 + i - W;
        const int rr = min(max(mirror(g, p.H) - p.in_row0, 0), p.in_rows - 1);
        const float* src = row_ptr(p, b, p.in_row0 + rr);
        const int gx = mirror(tx0 - W + c, p.Wd);
        GC_CHK(p, src + gx, 4);
        fv[u] = __ldg(src + gx);
      }
    }
#pragma unroll
    for (int u = 0; u < kFuSB; u++) {
      const int k = k0 + u * kFuThreads;
      if (k < C::NF) {
        float a, e;
        centre(p, fv[u], a, e);
        if (p.raw) { e = fv[u]; a = 0.f; }               // gc_gaussian: (f, 0)
        sF[k] = make_float2(e, e * a);
        sA2[k] = a * a;
      }
    }
  }
#pragma unroll
  for (int i = 0; i < C::RY; i++) {
    float e;
    centre(p, fo[i], av[i], e);
    pwx[i] = 1.f;                                       // G'_{2p} = a'^{2p}
    P[i] = Q[i] = vpy[i] = raw0[i] = 0.f;
  }
  __syncthreads();

  for (int pp = 0; pp < p.NP; pp++) {
    // 2. row pass over the region rows: RX consecutive tile columns per item, taps in ascending m
    for (int it = threadIdx.x; it < C::RH * (kFuTX / C::RX); it += kFuThreads) {
      const int r = it / (kFuTX / C::RX), c0 = (it % (kFuTX / C::RX)) * C::RX;
      const float2* src = sF + r * C::RW + c0;
      float2 acc[C::RX];
#pragma unroll
      for (int i = 0; i < C::RX; i++) acc[i] = make_float2(0.f, 0.f);
#pragma unroll
      for (int j = 0; j < C::RX + 2 * W; j++) {
        const float2 v = src[j];
#pragma unroll
        for (int i = 0; i < C::RX; i++) {
          const int m = j - i;
          if (m >= 0 && m <= 2 * W) acc[i] = f2fma(make_float2(p.tap[m], p.tap[m]), v, acc[i]);
        }
      }
#pragma unroll
      for (int i = 0; i < C::RX; i++) sR[r * kFuTX + c0 + i] = acc[i];
    }
    __syncthreads();
    // 3. column pass + eqs. (8)-(9) with v_n = chat_n G'_n:  Q += v_n Fbar_n,  P += v_{n-1} Fbar_n
    {
      float2 acc[C::RY];
#pragma unroll
      for (int i = 0; i < C::RY; i++) acc[i] = make_float2(0.f, 0.f);
#pragma unroll
      for (int j = 0; j < C::RY + 2 * W; j++) {
        const float2 v = sR[(i0 + j) * kFuTX + cx];
#pragma unroll
        for (int i = 0; i < C::RY; i++) {
          const int m = j - i;
          if (m >= 0 && m <= 2 * W) acc[i] = f2fma(make_float2(p.tap[m], p.tap[m]), v, acc[i]);
        }
      }
      if (pp == 0) {
#pragma unroll
        for (int i = 0; i < C::RY; i++) raw0[i] = acc[i].x;
      }
      const float2 c2 = p.chat2[pp];
#pragma unroll
      for (int i = 0; i < C::RY; i++) {
        const float v0 = c2.x * pwx[i];
        const float v1 = c2.y * (pwx[i] * av[i]);
        Q[i] = fmaf(v0, acc[i].x, Q[i]);
        Q[i] = fmaf(v1, acc[i].y, Q[i]);
        P[i] = fmaf(vpy[i], acc[i].x, P[i]);
        P[i] = fmaf(v0, acc[i].y, P[i]);
        vpy[i] = v1;
        pwx[i] *= av[i] * av[i];
      }
    }
    // 4. next plane pair: psi <- psi a'^2 over the region (the row pass of this pair is done)
    if (pp + 1 < p.NP) {
      for (int k = threadIdx.x; k < C::NF; k += kFuThreads) sF[k] = f2mul(sF[k], make_float2(sA2[k], sA2[k]));
    }
    __syncthreads();
  }

  // 5. eq. (10), uncentring and the guard
  unsigned nguard = 0;
  if (x < p.Wd) {
    float* out = p.out + b * p.out_img_stride + x;
#pragma unroll
    for (int i = 0; i < C::RY; i++) {
      const int yy = ty0 + i0 + i;
      if (yy >= p.out_rows) break;
      const float Qi = Q[i], Pi = P[i];
      float o;
      if (p.raw) {
        o = raw0[i];
      } else if (Qi > 0.f && isfinite(Qi) && isfinite(Pi)) {
        o = p.t_c + p.t_h * __fdividef(Pi, Qi);          // eq. (10) + uncentring
      } else {                                            // guard (R8)
        o = fminf(fmaxf(fo[i], p.L), p.U);
        nguard++;
      }
      GC_CHK(p, &out[(long long)yy * p.Wd], 4);
      out[(long long)yy * p.Wd] = o;
    }
  }
  count_guarded(p.fallback, 0xffffffffu, nguard);
}

template <int W, int TY>
cudaError_t launch_fused_t(const KParams& p, cudaStream_t s) {
  using C = FuCfg<W, TY>;
  auto k = k_fused_fir<W, TY>;
  static std::atomic<unsigned long long> ready{0};
  const cudaError_t e0 = once_per_device(ready, [&]() {
    return cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
  });
  if (e0 != cudaSuccess) return e0;
  const long long nt = (long long)((p.Wd + kFuTX - 1) / kFuTX) * ((p.out_rows + TY - 1) / TY) * p.B;
  if (p.ev[0]) cudaEventRecord(p.ev[0], s);
  k<<<(unsigned)nt, kFuThreads, C::SMEM, s>>>(p);
  const cudaError_t e = cudaGetLastError();
  // (one kernel: the instrumented "row" interval is the whole filter, the "column" one empty)
  if (p.ev[1]) cudaEventRecord(p.ev[1], s);
  if (p.ev[2]) cudaEventRecord(p.ev[2], s);
  return e;
}

template <int W>
struct FuTable {
  static cudaError_t go(const KParams& p, bool tall, cudaStream_t s) {
    if (p.R == W) return tall ? launch_fused_t<W, 32>(p, s) : launch_fused_t<W, 16>(p, s);
    return FuTable<W - 1>::go(p, tall, s);
  }
};
template <>
struct FuTable<0> {
  static cudaError_t go(const KParams&, bool, cudaStream_t) { return cudaErrorInvalidValue; }
};

}  // namespace

// The fused path takes the FIR's small calls: W <= kFuMaxW and at most kFuMaxPx output pixels
// (GC_FIR_FUSED=0 / 1 forces the two-pass / the fused path where W allows, for A/B and tests).
bool fused_fir_applies(const KParams& p) {
  static const int force = [] {
    const char* v = std::getenv("GC_FIR_FUSED");
    return v ? std::atoi(v) : -1;
  }();
  if (p.fp64 || p.op != GC_OP_FIR || p.R < 1 || p.R > kFuMaxW) return false;
  if (force >= 0) return force != 0;
  return (long long)p.B * p.out_rows * p.Wd <= kFuMaxPx;
}

cudaError_t launch_fused_fir(const KParams& p, cudaStream_t s) {
  // 32-row tiles unless that leaves SMs idle (then 16-row tiles: twice the CTAs)
  const long long t32 = (long long)((p.Wd + kFuTX - 1) / kFuTX) * ((p.out_rows + 31) / 32) * p.B;
  return FuTable<kFuMaxW>::go(p, t32 >= p.num_sms, s);
}

}  // namespace gc
