// gc_device.cuh — small device helpers shared by the sm_100a kernels.
#pragma once

#include <cuda_runtime.h>

#include "gc_internal.h"

namespace gc {

// Packed fp32x2 arithmetic (SASS FFMA2 / FMUL2): one issue slot for two FP32 lanes.
// Measured on B200: the FMA pipe stays at 128 lanes/clk/SM, so FFMA2 halves issue
// pressure without raising the FMA peak (profiles/r01_ubench_fp32.txt).
__device__ __forceinline__ float2 f2fma(float2 a, float2 b, float2 c) {
  float2 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(*reinterpret_cast<unsigned long long*>(&d))
      : "l"(*reinterpret_cast<const unsigned long long*>(&a)),
        "l"(*reinterpret_cast<const unsigned long long*>(&b)),
        "l"(*reinterpret_cast<const unsigned long long*>(&c)));
  return d;
}

__device__ __forceinline__ float2 f2mul(float2 a, float2 b) {
  float2 d;
  asm("mul.rn.f32x2 %0, %1, %2;"
      : "=l"(*reinterpret_cast<unsigned long long*>(&d))
      : "l"(*reinterpret_cast<const unsigned long long*>(&a)),
        "l"(*reinterpret_cast<const unsigned long long*>(&b)));
  return d;
}

__device__ __forceinline__ float2 f2add(float2 a, float2 b) {
  float2 d;
  asm("add.rn.f32x2 %0, %1, %2;"
      : "=l"(*reinterpret_cast<unsigned long long*>(&d))
      : "l"(*reinterpret_cast<const unsigned long long*>(&a)),
        "l"(*reinterpret_cast<const unsigned long long*>(&b)));
  return d;
}

__device__ __forceinline__ float2 f2sub(float2 a, float2 b) {
  float2 d;
  asm("sub.rn.f32x2 %0, %1, %2;"
      : "=l"(*reinterpret_cast<unsigned long long*>(&d))
      : "l"(*reinterpret_cast<const unsigned long long*>(&a)),
        "l"(*reinterpret_cast<const unsigned long long*>(&b)));
  return d;
}

__device__ __forceinline__ float2 f2s(float s) { return make_float2(s, s); }

// Programmatic dependent launch (PDL): the column pass is launched while the row pass
// drains; it waits here (all of the row pass complete and visible) before reading planes.
// Both are no-ops when the launch did not use the PDL attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Guard counter (R8): one atomic per warp instead of one per guarded pixel.
// Every lane of `mask` must call it (lanes outside it are not counted).
__device__ __forceinline__ void count_guarded(unsigned long long* ctr, unsigned mask, unsigned n) {
  if (!ctr) return;
  const unsigned tot = __reduce_add_sync(mask, n);
  if (tot && (threadIdx.x & 31) == (unsigned)(__ffs(mask) - 1)) atomicAdd(ctr, (unsigned long long)tot);
}

// Whole-sample symmetric extension (R5): period 2n-2, n = 1 -> 0.
static __device__ __noinline__ int mirror_slow(int p, int n) {
  if (n <= 1) return 0;
  const int period = 2 * n - 2;
  p = p < 0 ? -p : p;
  p %= period;
  return p < n ? p : period - p;
}
__device__ __forceinline__ int mirror(int p, int n) {
  return (unsigned)p < (unsigned)n ? p : mirror_slow(p, n);   // interior: no arithmetic
}

// 2^x on the MUFU (one instruction; denormal results flush to 0, which only occurs for
// e = exp(-g^2/2sr^2) < 2^-126, i.e. terms far below fp32 resolution of the sums).
__device__ __forceinline__ float ex2_ftz(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// ---- bounds checks of the GC_BOUNDS_CHECK build (libgc_check.so; compute-sanitizer is not
// available on the B200 pool): [ptr, ptr + bytes) must lie in an input segment (of some image of
// the batch), the plane / scratch buffer, the output, or the taps; otherwise the access is counted
// in *p.oob.  GC_CHK compiles to nothing in the product library.
#ifdef GC_BOUNDS_CHECK
static __device__ __noinline__ void gc_oob_note(const KParams& p) {
  if (p.oob) atomicAdd(p.oob, 1ull);
}
__device__ __forceinline__ bool gc_in(const void* ptr, size_t n, const void* base, size_t bytes) {
  const char* a = reinterpret_cast<const char*>(ptr);
  const char* b = reinterpret_cast<const char*>(base);
  return base && a >= b && a + n <= b + bytes;
}
__device__ __forceinline__ void gc_chk(const KParams& p, const void* ptr, size_t n) {
  if (gc_in(ptr, n, p.planes, p.planes_bytes)) return;
  if (gc_in(ptr, n, p.out, (size_t)p.B * p.out_img_stride * 4)) return;
  if (p.taps_g && gc_in(ptr, n, p.taps_g, (size_t)(2 * p.R + 1) * 16)) return;
  for (int k = 0; k < 3; k++) {
    if (p.seg[k].rows <= 0) continue;
    const size_t img = (size_t)p.seg[k].rows * p.Wd * 4;
    for (int b = 0; b < p.B; b++)
      if (gc_in(ptr, n, p.seg[k].ptr + (long long)b * p.seg_img_stride, img)) return;
  }
  gc_oob_note(p);
}
#define GC_CHK(p, ptr, n) gc_chk((p), (ptr), (n))
#else
#define GC_CHK(p, ptr, n) ((void)0)
#endif

// Pointer to global row gy of image b, found in the input segments.
__device__ __forceinline__ const float* row_ptr(const KParams& p, int b, int gy) {
#pragma unroll
  for (int k = 0; k < 3; k++) {
    const int r = gy - p.seg[k].row0;
    if (r >= 0 && r < p.seg[k].rows) return p.seg[k].ptr + b * p.seg_img_stride + (long long)r * p.Wd;
  }
  return p.seg[0].ptr + b * p.seg_img_stride;  // unreachable after host validation
}

// Pointer to global row gy of image b if rows gy .. gy+n-1 all lie in one input segment
// (consecutive rows then sit Wd floats apart), else nullptr.
__device__ __forceinline__ const float* row_run_ptr(const KParams& p, int b, int gy, int n) {
#pragma unroll
  for (int k = 0; k < 3; k++) {
    const int r = gy - p.seg[k].row0;
    if (r >= 0 && r + n <= p.seg[k].rows) return p.seg[k].ptr + b * p.seg_img_stride + (long long)r * p.Wd;
  }
  return nullptr;
}

// Eq. (17) centring and the scaled auxiliary variable a' = g / t_h in [-1, 1], plus the
// Gaussian factor e = exp(-g^2 / 2 sigma_r^2) of eq. (6), as exp2(ex_k a'^2).
__device__ __forceinline__ void centre(const KParams& p, float f, float& a, float& e) {
  f = fminf(fmaxf(f, p.L), p.U);            // inputs clamped to [L, U] (R7)
  a = (f - p.t_c) * p.inv_th;
  e = ex2_ftz(p.ex_k * (a * a));
}

// a' alone (the recombination of eqs. (8)-(9) needs no Gaussian factor).
__device__ __forceinline__ float centre_a(const KParams& p, float f) {
  f = fminf(fmaxf(f, p.L), p.U);
  return (f - p.t_c) * p.inv_th;
}

}  // namespace gc
