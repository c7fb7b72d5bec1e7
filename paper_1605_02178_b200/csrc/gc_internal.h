// gc_internal.h — declarations shared by the C ABI (gc_api.cpp) and the sm_100a
// kernels (gc_fir.cu).  Not part of the public ABI.
#pragma once

#include <cstdint>

#include "../../include/gc.h"

#include <cuda_runtime.h>

namespace gc {

// Host coefficient cache (gc_coeffs.cpp): c_n (eq. 19) and the normalised c_n mu^n.
gc_status coeffs_cached(int N, double sigma_r, double L, double U, const double** c,
                        const double** cmu, double* mu);

constexpr int kMaxPlanes = GC_N_MAX + 2 + 1;   // N+2 planes, rounded up to even
constexpr int kMaxPairs = (kMaxPlanes + 1) / 2;
constexpr int kMaxTemplW = 24;                 // FIR radius range with unrolled kernels
constexpr int kMaxFirW = 1024;                 // runtime-W FIR kernels (taps in global)

// One input-row segment (device pointer to rows [row0, row0+rows) of the global image).
struct Seg {
  const float* ptr;
  int row0;
  int rows;
};

// Everything a launch needs; passed by value (param space / constant bank 0).
struct KParams {
  int H;                  // global image rows (symmetric extension at 0 and H-1)
  int Wd;                 // image width (symmetric extension at 0 and Wd-1)
  int B;                  // images in the batch (grid.z)
  int R;                  // spatial radius W_s = ceil(3 sigma_s)
  int NP;                 // plane pairs: planes 0 .. 2NP-1 (>= N+2, padded to even)
  int in_row0, in_rows;   // global rows held by the plane buffer
  int out_row0, out_rows; // global rows written
  Seg seg[3];             // input rows (see gc_filter_window)
  long long seg_img_stride;   // elements between consecutive images in every segment
  float2* planes;         // row pass output [B][NP][in_rows][Wd] (plane pairs, row-major)
  int in_pitch;           // unused (reserved)
  unsigned* counters;     // device scratch: dynamic task counters (zeroed on device)
  long long planes_img_stride; // float2 elements per image
  float* out;             // [B][out_rows][Wd]
  long long out_img_stride;
  float L, U;             // clamp range
  float t_c;              // (L+U)/2                        eq. (17)
  float t_h;              // (U-L)/2  (output scale: sigma_r sqrt(mu))
  float inv_th;           // 1/t_h   (a' = g / t_h in [-1, 1])
  float ex_k;             // -mu/2 * log2(e):  exp(-g^2/2sr^2) = exp2(ex_k a'^2)
  unsigned long long* fallback;  // may be null
  const float2* taps_g;   // (k_m, k_m), m = 0..2R, in global memory (runtime-W kernels)
  cudaEvent_t ev[3];      // optional timing events (host side only; not read on device)
  float2 chat2[kMaxPairs];         // (chat_{2p}, chat_{2p+1}), zero beyond N
  float tap[2 * kMaxTemplW + 1];   // k_m, m = 0..2R (unrolled kernels; FFMA2 scalar broadcast)
  int ctas_per_sm;                 // persistent-grid sizing (host side)
  int num_sms;
};

// Launch the two-pass FIR pipeline (row pass + column pass with recombination) on
// `stream`.  Scratch (the plane buffer) must already be in p.planes.
cudaError_t launch_fir_two_pass(const KParams& p, cudaStream_t stream);

}  // namespace gc
