// gc_fp64.cu — the GCF hot path in binary64 internal arithmetic.
//
// At the (sigma_r, N) BASELINE.json states, eq. (19)'s coefficients make the recombination of
// eqs. (8)-(9) cancel by up to 10^66 (R1): the fp32 path cannot follow the
// fp64 oracle there.  This mode runs the same pipeline — centring (eq. 17), auxiliary planes
// (eq. 6), the truncated separable FIR of eq. (7) and eqs. (8)-(10) with the guard of R8 — with
// every intermediate in binary64 (input and output stay fp32), so the stated configs can be
// checked against the oracle element by element.  Plain one-thread-per-output kernels: FP64
// runs at half the FP32 rate on B200 and this mode is a correctness instrument, not the
// throughput path.
#include <atomic>

#include "gc_device.cuh"

namespace gc {

constexpr int kF64TX = 64, kF64TY = 4;

__device__ __forceinline__ void centre_d(const KParams& p, float f, double& a, double& e) {
  const double x = fmin(fmax((double)f, p.d_L), p.d_U);
  a = (x - p.d_tc) * p.d_inv_th;
  e = exp(p.d_exk * (a * a));
}

// Row pass: TY rows x TX outputs per CTA; the current plane pair of the staged row segment is
// advanced in shared memory (psi <- psi a'^2) between pairs.
__global__ void __launch_bounds__(256) k_row_f64(const KParams p) {
  pdl_trigger();
  extern __shared__ double2 smem_f64[];
  const int R = p.R;
  const int SW = kF64TX + 2 * R;
  double2* sPL = smem_f64;                               // [TY][SW] current plane pair
  double* sA2 = reinterpret_cast<double*>(sPL + kF64TY * SW);   // [TY][SW] a'^2
  const int b = blockIdx.z, x0 = blockIdx.x * kF64TX, r0 = blockIdx.y * kF64TY;
  const int tid = threadIdx.x;
  for (int r = 0; r < kF64TY; r++) {
    const int rr = r0 + r;
    if (rr >= p.in_rows) break;
    const float* src = row_ptr(p, b, p.in_row0 + rr);
    for (int c = tid; c < SW; c += 256) {
      double a, e;
      GC_CHK(p, src + mirror(x0 - R + c, p.Wd), 4);
      centre_d(p, __ldg(src + mirror(x0 - R + c, p.Wd)), a, e);
      sPL[r * SW + c] = make_double2(e, e * a);
      sA2[r * SW + c] = a * a;
    }
  }
  __syncthreads();
  const int r = tid / kF64TX, xo = tid % kF64TX;
  const int rr = r0 + r;
  const bool ok = rr < p.in_rows && x0 + xo < p.Wd;
  const long long pstride = (long long)p.in_rows * p.Wd;
  double2* planes = reinterpret_cast<double2*>(p.planes);
  for (int pp = 0; pp < p.NP; pp++) {
    if (ok) {
      double ax = 0.0, ay = 0.0;
      for (int m = 0; m <= 2 * R; m++) {
        const double2 v = sPL[r * SW + xo + m];
        const double k = p.taps_d[m];
        ax = fma(k, v.x, ax);
        ay = fma(k, v.y, ay);
      }
      GC_CHK(p, &planes[b * p.planes_img_stride + pp * pstride + (long long)rr * p.Wd + x0 + xo], 16);
      planes[b * p.planes_img_stride + pp * pstride + (long long)rr * p.Wd + x0 + xo] = make_double2(ax, ay);
    }
    __syncthreads();
    for (int idx = tid; idx < kF64TY * SW; idx += 256) {
      const double w = sA2[idx];
      sPL[idx] = make_double2(sPL[idx].x * w, sPL[idx].y * w);
    }
    __syncthreads();
  }
}

// Column pass + eqs. (8)-(10): one output pixel per thread.
__global__ void __launch_bounds__(256) k_col_f64(const KParams p) {
  pdl_wait();
  const int b = blockIdx.z;
  const int x = blockIdx.x * 32 + threadIdx.x % 32;
  const int y = blockIdx.y * 8 + threadIdx.x / 32;
  const bool live = x < p.Wd && y < p.out_rows;
  unsigned guarded = 0;
  if (live) {
    const int R = p.R;
    const int gy = p.out_row0 + y;
    GC_CHK(p, row_ptr(p, b, gy) + x, 4);
    const float f = __ldg(row_ptr(p, b, gy) + x);
    double a, e;
    centre_d(p, f, a, e);
    const long long pstride = (long long)p.in_rows * p.Wd;
    const double2* planes = reinterpret_cast<const double2*>(p.planes) + b * p.planes_img_stride + x;
    double P = 0.0, Q = 0.0, G = 1.0, vprev = 0.0;
    for (int pp = 0; pp < p.NP; pp++) {
      const double2* pl = planes + pp * pstride;
      double fx = 0.0, fy = 0.0;                          // (Fbar'_{2p}, Fbar'_{2p+1})
      for (int m = 0; m <= 2 * R; m++) {
        const int q = mirror(gy + m - R, p.H) - p.in_row0;
        GC_CHK(p, &pl[(long long)q * p.Wd], 16);
        const double2 v = pl[(long long)q * p.Wd];
        fx = fma(p.taps_d[m], v.x, fx);
        fy = fma(p.taps_d[m], v.y, fy);
      }
      // eqs. (8)-(9), ascending n:  Q += v_n Fbar_n,  P += v_{n-1} Fbar_n,  v_n = chat_n a'^n
      const double v0 = p.chat_d[2 * pp] * G;
      const double v1 = p.chat_d[2 * pp + 1] * (G * a);
      Q = fma(v0, fx, Q);
      P = fma(vprev, fx, P);
      Q = fma(v1, fy, Q);
      P = fma(v0, fy, P);
      vprev = v1;
      G *= a * a;
    }
    float o;
    if (Q > 0.0 && isfinite(Q) && isfinite(P)) {
      o = (float)(p.d_tc + p.d_th * (P / Q));               // eq. (10) + uncentring
    } else {                                                // guard (R8)
      o = (float)fmin(fmax((double)f, p.d_L), p.d_U);
      guarded = 1;
    }
    GC_CHK(p, &p.out[b * p.out_img_stride + (long long)y * p.Wd + x], 4);
    p.out[b * p.out_img_stride + (long long)y * p.Wd + x] = o;
  }
  count_guarded(p.fallback, __activemask(), guarded);
}

cudaError_t launch_fp64_two_pass(const KParams& p, cudaStream_t s) {
  const size_t smem = (size_t)kF64TY * (kF64TX + 2 * p.R) * (sizeof(double2) + sizeof(double));
  static std::atomic<unsigned long long> ready{0};
  cudaError_t e = once_per_device(ready, [&]() {   // the largest radius's size: covers every call
    return cudaFuncSetAttribute(k_row_f64, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)((size_t)kF64TY * (kF64TX + 2 * kMaxFirW) * (sizeof(double2) + sizeof(double))));
  });
  if (e != cudaSuccess) return e;
  if (p.ev[0]) cudaEventRecord(p.ev[0], s);
  dim3 gr((p.Wd + kF64TX - 1) / kF64TX, (p.in_rows + kF64TY - 1) / kF64TY, p.B);
  k_row_f64<<<gr, 256, smem, s>>>(p);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (p.ev[1]) cudaEventRecord(p.ev[1], s);
  dim3 gc((p.Wd + 31) / 32, (p.out_rows + 7) / 8, p.B);
  e = launch_k(k_col_f64, gc, dim3(256), 0, s, p.ev[1] == nullptr, p);
  if (p.ev[2]) cudaEventRecord(p.ev[2], s);
  return e;
}

}  // namespace gc
