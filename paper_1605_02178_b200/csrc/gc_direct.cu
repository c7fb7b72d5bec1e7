// gc_direct.cu — the direct bilateral filter of eq. (1) on sm_100a (SURVEY §8(f)
// NEXT-3): the O(sigma_s^2) reference the GCF approximates, used for full-image MSE / PSNR of
// the fast filter at sizes the CPU oracle cannot reach.
//
//   B[f](i) = sum_{j in Omega} g_s(j) g_r(f(i-j) - f(i)) f(i-j) / sum_{j in Omega} g_s(j) g_r(...)
//
// Omega = [-W, W]^2, W = ceil(3 sigma_s) (R4), whole-sample symmetric
// extension (R5), spatial taps unnormalised (the normalisation cancels, R6).  Each tap
// costs one MUFU ex2: w = 2^(cr d^2 + cs (mx^2 + my^2)), so the kernel is bound by the MUFU
// pipe (16 lanes/clk/SM), not by memory: the (2W+1)^2 reads per output hit L1.
//
// One thread per output pixel; 32 x 8 outputs per CTA.  Per window row the thread keeps a
// row-partial numerator / denominator and adds it to the total once (fp32 rounding grows with
// 2W+1, not (2W+1)^2).
#include "gc_device.cuh"

namespace gc {

struct DirectParams {
  const float* img;
  float* out;
  int B, H, Wd, R;
  long long img_stride;
  float cr;   // -log2(e) / (2 sigma_r^2)
  float cs;   // -log2(e) / (2 sigma_s^2)
};

__global__ void __launch_bounds__(256) k_direct(const DirectParams d) {
  const int b = blockIdx.z;
  const int x = blockIdx.x * 32 + (threadIdx.x & 31);
  const int y = blockIdx.y * 8 + (threadIdx.x >> 5);
  if (x >= d.Wd || y >= d.H) return;
  const float* img = d.img + b * d.img_stride;
  const float fi = __ldg(img + (long long)y * d.Wd + x);
  const int R = d.R;
  float num = 0.f, den = 0.f;
  for (int my = -R; my <= R; my++) {
    const float* row = img + (long long)mirror(y + my, d.H) * d.Wd;
    const float ty = d.cs * (float)(my * my);
    float rn = 0.f, rd = 0.f;
    const bool xin = x - R >= 0 && x + R < d.Wd;
    if (xin) {
      const float* rp = row + x - R;
#pragma unroll 4
      for (int k = 0; k <= 2 * R; k++) {
        const int mx = k - R;
        const float fj = __ldg(rp + k);
        const float df = fj - fi;
        const float w = ex2_ftz(fmaf(d.cr * df, df, fmaf(d.cs, (float)(mx * mx), ty)));
        rn = fmaf(w, fj, rn);
        rd += w;
      }
    } else {
      for (int mx = -R; mx <= R; mx++) {
        const float fj = __ldg(row + mirror(x + mx, d.Wd));
        const float df = fj - fi;
        const float w = ex2_ftz(fmaf(d.cr * df, df, fmaf(d.cs, (float)(mx * mx), ty)));
        rn = fmaf(w, fj, rn);
        rd += w;
      }
    }
    num += rn;
    den += rd;
  }
  d.out[b * d.img_stride + (long long)y * d.Wd + x] = num / den;   // den >= w(0,0) = 1
}

cudaError_t launch_direct(const float* img, int B, int H, int W, int R, float sigma_s, float sigma_r, float* out,
                          cudaStream_t s) {
  DirectParams d;
  d.img = img;
  d.out = out;
  d.B = B;
  d.H = H;
  d.Wd = W;
  d.R = R;
  d.img_stride = (long long)H * W;
  d.cr = (float)(-1.4426950408889634 / (2.0 * (double)sigma_r * (double)sigma_r));
  d.cs = (float)(-1.4426950408889634 / (2.0 * (double)sigma_s * (double)sigma_s));
  dim3 grid((W + 31) / 32, (H + 7) / 8, B);
  k_direct<<<grid, 256, 0, s>>>(d);
  return cudaGetLastError();
}

// Positive control of the GC_BOUNDS_CHECK machinery (gc_debug_oob_selftest): GC_CHK of one
// address just past a region and one inside it; only the first may be counted.  No memory is
// accessed.
__global__ void k_oob_selftest(const KParams p) {
  if (threadIdx.x == 0) {
    GC_CHK(p, reinterpret_cast<const char*>(p.planes) + p.planes_bytes, 1);   // one byte past the end
    GC_CHK(p, p.planes, 8);                                                      // inside
  }
}

cudaError_t launch_oob_selftest(const KParams& p, cudaStream_t s) {
  k_oob_selftest<<<1, 32, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace gc
