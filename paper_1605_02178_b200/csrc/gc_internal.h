// gc_internal.h — declarations shared by the C ABI (gc_api.cpp) and the sm_100a
// kernels (gc_fir.cu).  Not part of the public ABI.
#pragma once

#include <atomic>
#include <cstdint>
#include <utility>
#include <vector>

#include "../../include/gc.h"

#include <cuda_runtime.h>

namespace gc {

// Host coefficient cache (gc_coeffs.cpp): c_n (eq. 19) and the normalised c_n mu^n.
// Copies out of a bounded LRU memo (gc_lru.h); c / cmu / mu may be null.
gc_status coeffs_cached(int N, double sigma_r, double L, double U, std::vector<double>* c,
                        std::vector<double>* cmu, double* mu);

// Stream-ordered scratch from libgc's private per-device pool (gc_api.cpp); free with cudaFreeAsync.
cudaError_t scratch_alloc(void** ptr, size_t bytes, cudaStream_t s);
// GC_BOUNDS_CHECK builds: device counter of out-of-bounds accesses (nullptr otherwise).
unsigned long long* oob_counter();

constexpr int kMaxPlanes = GC_N_MAX + 2 + 1;   // N+2 planes, rounded up to even
constexpr int kMaxPairs = (kMaxPlanes + 1) / 2;
constexpr int kMaxTemplW = 24;                 // FIR radius range with unrolled kernels
constexpr int kMaxFirW = 1024;                 // runtime-W FIR kernels (taps in global)
constexpr int kO1K = 5;                        // O(1) operator: cosine terms (q = 0 is the box); free-frequency fit
constexpr int kO1MaxW = 4096;                  // O(1) operator radius limit
constexpr int kO1AutoMinW = kMaxTemplW + 1;     // GC_OP_AUTO: FIR for W <= 24 (unrolled kernels), O(1) above

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
  int op;                 // resolved operator: GC_OP_FIR or GC_OP_O1 (host side)
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
  // GC_BOUNDS_CHECK builds (libgc_check.so): every global access of the kernels is checked against
  // the buffers below and violations are counted in *oob (gc_debug_oob_count); null otherwise
  unsigned long long* oob;
  size_t planes_bytes;    // bytes of the plane buffer (incl. counters and the Deriche scratch)
  const float2* taps_g;   // (k_m, k_m), m = 0..2R, in global memory (runtime-W kernels)
  cudaEvent_t ev[3];      // optional timing events (host side only; not read on device)
  float2 chat2[kMaxPairs];         // (chat_{2p}, chat_{2p+1}), zero beyond N
  float tap[2 * kMaxTemplW + 1];   // k_m, m = 0..2R (unrolled kernels; FFMA2 scalar broadcast)
  int ctas_per_sm;                 // persistent-grid sizing (host side)
  int num_sms;
  // O(1) exact-window operator (gc_o1.cu): k_m ~ sum_q alpha_q cos(w_q m) on |m| <= W
  float o1_alpha[kO1K];            // alpha_q (q = 0: box term)
  float o1_nk[kO1K];               // -4 sin^2(w_q / 2)   (Reinsch form of the resonator)
  float o1_a[kO1K];                // alpha_q cos(w_q W)        (alpha folded into the states)
  float o1_nb[kO1K];               // -alpha_q cos(w_q (W + 1))
  int o1_seg_x, o1_nseg_x;         // row pass: x-segment length (multiple of 32) and count
  int o1_seg_y, o1_nseg_y;         // column pass: y-segment length and count
  int o1_groups;                   // row pass: plane-pair groups (<= 4 pairs each)
  int o1_stages;                   // pair-parallel column pass: TMA ring stages
  // direct lead-in (row pass): for s = 0..2W, m = s - W, two float4 per s:
  // {alpha_q cos(w_q m)}_{q=1..4} and {alpha_q (cos(w_q m) - cos(w_q (m+1)))} (the m = W entry
  // without its cos(w_q (W+1)) term); null = lead the recursion in from a zero state instead
  const float4* o1_lead;
  int raw;                         // 1: eq. (7) of f itself (gc_gaussian): pair 0 = (f, 0), out = Fbar_0
  // Deriche-class recursive operator (gc_deriche.cu; GC_OP_DERICHE): two 2nd-order sections per
  // direction, 1/Z folded into b0, b1, c1, c2
  float dr_b0[2], dr_b1[2], dr_c1[2], dr_c2[2], dr_a1[2], dr_a2[2];
  int dr_K;                        // mirror padding / lead-in per side: ceil(10 sigma_s)
  int dr_seg_x, dr_nseg_x;         // row pass: x-segment length (multiple of 8) and count
  int dr_seg_y, dr_nseg_y;         // column pass: y-segment length and count
  float2* scratch;                 // causal partial sums (as large as the plane buffer)
  // binary64 internal arithmetic (gc_fp64.cu; gc_params.precision = GC_PREC_FP64)
  int fp64;
  float sigma_s_host;                             // sigma_s (host side: taps)
  double d_tc, d_th, d_inv_th, d_exk, d_L, d_U;   // d_exk = -mu/2 (natural exp)
  const double* taps_d;                           // k_m, m = 0..2R (device)
  double chat_d[kMaxPlanes];                      // chat_n, zero beyond N
};

// O(1) operator constants for radius R = ceil(3 sigma_s) (gc_api.cpp): least-squares K-term
// cosine expansion of the truncated taps on |m| <= R, half-period Lh searched for the smallest
// max error.  alpha/omega in binary64; fit_err = max_m |expansion - k_m|.
struct O1Fit {
  int R;
  double Lh;
  double alpha[kO1K];
  double omega[kO1K];
  double fit_err;
};
O1Fit o1_fit_cached(float sigma_s);

// O(1) column pass: G lanes per column share the NP plane pairs, npg = ceil(NP / G) <= 7 each
// (G = 1 up to 7 pairs: one lane holds every pair of its column, no cross-lane reduction).
inline void o1_col_split(int NP, int& G, int& npg) {
  G = NP <= 7 ? 1 : NP <= 14 ? 2 : NP <= 28 ? 4 : 8;
  npg = (NP + G - 1) / G;
}

// Segments of a line of `len` samples for `base` independent lines (tasks = base x segments),
// each segment paying a lead-in of `lead` samples, on a GPU that holds `resident` warps at once:
// the count minimising waves x (segment + lead-in), i.e. the last wave's tail against the
// lead-in overhead (O(1) and Deriche passes; measured on B200 in profiles/r01_ab_experiments.md).
// Segments are multiples of `align` samples.
inline void pick_segments(int len, long long base, int lead, long long resident, int align, int& seg, int& nseg) {
  resident = resident < 1 ? 1 : resident;
  int nmax = len / (lead < 1 ? 1 : lead);
  nmax = nmax < 1 ? 1 : (nmax > 256 ? 256 : nmax);
  double best = 0;
  seg = (len + align - 1) / align * align;
  nseg = 1;
  for (int n = 1; n <= nmax; n++) {
    const int sg = ((len + n - 1) / n + align - 1) / align * align;
    const int nn = (len + sg - 1) / sg;
    const long long waves = (base * nn + resident - 1) / resident;
    const double t = (double)waves * (double)(sg + lead);
    if (n == 1 || t < best * 0.999) {
      best = t;
      seg = sg;
      nseg = nn;
    }
  }
}

// Per-device one-time setup (function attributes are per device context): run fn once per
// (call site, device); fn must be idempotent (two threads may both run it once).
template <typename F>
cudaError_t once_per_device(std::atomic<unsigned long long>& done, F&& fn) {
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess) return cudaErrorInvalidDevice;
  const unsigned long long bit = 1ull << (d & 63);
  if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
  const cudaError_t e = fn();
  if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
  return e;
}

// Launch `kernel` on `s`; with pdl = true the launch carries the programmatic-stream-
// serialization attribute (its prologue overlaps the previous kernel's tail; the kernel
// calls pdl_wait() before consuming that kernel's output).
template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, bool pdl,
                     Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// Launch the two-pass FIR pipeline (row pass + column pass with recombination) on
// `stream`.  Scratch (the plane buffer) must already be in p.planes.
cudaError_t launch_fir_two_pass(const KParams& p, cudaStream_t stream);
// Small-image FIR path (gc_fused.cu): one launch, both passes of eq. (7) in shared memory per tile
constexpr int kFuMaxW = kMaxTemplW;
constexpr long long kFuMaxPx = GC_FUSED_MAX_PX;  // output pixels per call (B x rows x width)
bool fused_fir_applies(const KParams& p);
cudaError_t launch_fused_fir(const KParams& p, cudaStream_t stream);

// Launch the two-pass O(1) exact-window pipeline (gc_o1.cu).  Same buffers and semantics.
cudaError_t launch_o1_two_pass(const KParams& p, cudaStream_t stream);

// Two-pass Deriche-class recursive pipeline (gc_deriche.cu), NP <= kDrMaxPairs; p.scratch set.
constexpr int kDrMaxPairs = 8;
void deriche_constants(float sigma_s, KParams& k);
cudaError_t launch_deriche_two_pass(const KParams& p, cudaStream_t stream);

// Two-pass FIR pipeline in binary64 (gc_fp64.cu): planes are double2 pairs (twice the bytes).
cudaError_t launch_fp64_two_pass(const KParams& p, cudaStream_t stream);

// GC_BOUNDS_CHECK positive control (gc_direct.cu): counts exactly one out-of-bounds access.
cudaError_t launch_oob_selftest(const KParams& p, cudaStream_t s);

// Direct bilateral filter of eq. (1) (gc_direct.cu).
cudaError_t launch_direct(const float* img, int B, int H, int W, int R, float sigma_s, float sigma_r, float* out,
                          cudaStream_t s);

}  // namespace gc
