// gc_api.cpp — the C ABI of libgc (include/gc.h): argument validation, coefficient and
// tap preparation, stream-ordered scratch, and dispatch to the sm_100a kernels.
//
// Every step of the filter runs in the kernels of gc_fir.cu; this file only marshals
// arguments.  There is no CPU fallback: if the device path cannot run, the call fails
// with a status code.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <mutex>
#include <vector>

#include "gc_internal.h"

namespace gc {
namespace {

bool finite_pos(double x) { return std::isfinite(x) && x > 0; }

bool overlap(const void* a, size_t na, const void* b, size_t nb) {
  auto pa = reinterpret_cast<uintptr_t>(a), pb = reinterpret_cast<uintptr_t>(b);
  return pa < pb + nb && pb < pa + na;
}

// W_s = ceil(3 sigma_s) (R4)
int radius_of(float sigma_s) { return (int)std::ceil(3.0 * (double)sigma_s); }

// Rows of input a window's output rows depend on, per side: W_s for eq. (7), the lead-in /
// padding K = ceil(10 sigma_s) for the Deriche operator.
int halo_of(const gc_params* p) {
  return p->op == GC_OP_DERICHE ? (int)std::ceil(10.0 * (double)p->sigma_s) : radius_of(p->sigma_s);
}

// Truncated, normalised spatial taps k_m = exp(-m^2 / 2 sigma_s^2) / sum, |m| <= R (eq. 7).
std::vector<double> taps_of(float sigma_s, int R) {
  std::vector<double> k(2 * R + 1);
  double s = 0;
  const double ss = (double)sigma_s;
  for (int m = -R; m <= R; m++) s += (k[m + R] = std::exp(-(double)m * m / (2.0 * ss * ss)));
  for (auto& v : k) v /= s;
  return k;
}

// Constants of the O(1) exact-window operator (gc_o1.cu, gc_operator.cpp).
void o1_constants(float sigma_s, KParams& k) {
  const O1Fit f = o1_fit_cached(sigma_s);
  for (int q = 0; q < kO1K; q++) {
    const double w = f.omega[q];
    const double sh = std::sin(0.5 * w);
    // alpha_q folded into the recursion inputs (gc_o1.cu: the states are alpha_q S_q)
    k.o1_alpha[q] = (float)f.alpha[q];
    k.o1_nk[q] = (float)(-4.0 * sh * sh);
    k.o1_a[q] = (float)(f.alpha[q] * std::cos(w * f.R));
    k.o1_nb[q] = (float)(-f.alpha[q] * std::cos(w * (f.R + 1)));
  }
}

// Direct lead-in table of the row pass (KParams::o1_lead): the window sums of the alpha-folded
// resonator states at a segment's first output, written out as dot products with the taps
// alpha_q cos(w_q m) of the fit.  Empty when GC_O1_DIRECT_LEAD=0 (recursion lead-in, A/B).
std::vector<float4> o1_lead_table(float sigma_s, int W) {
  static const bool on = [] {
    const char* v = std::getenv("GC_O1_DIRECT_LEAD");
    return !(v && v[0] == '0');
  }();
  if (!on) return {};
  const O1Fit f = o1_fit_cached(sigma_s);
  if (f.R != W) return {};
  static_assert(kO1K == 5, "the lead-in table packs the 4 resonators into one float4");
  const int R = f.R;
  std::vector<float4> t(2 * (2 * R + 1));
  for (int s = 0; s <= 2 * R; s++) {
    const int m = s - R;
    double c[4], d[4];
    for (int q = 0; q < 4; q++) {
      const double a = f.alpha[q + 1], w = f.omega[q + 1];
      c[q] = a * std::cos(w * m);
      // D = S(x) - S(x-1) of the zero-extended signal: tap m of the window at x minus tap m+1
      // of the window at x-1 (which ends at m = W)
      d[q] = m < R ? a * (std::cos(w * m) - std::cos(w * (m + 1))) : c[q];
    }
    t[2 * s] = make_float4((float)c[0], (float)c[1], (float)c[2], (float)c[3]);
    t[2 * s + 1] = make_float4((float)d[0], (float)d[1], (float)d[2], (float)d[3]);
  }
  return t;
}

gc_status validate_params(const gc_params* p) {
  if (!p) return GC_EINVAL;
  if (p->N < 0) return GC_EINVAL;
  if (p->N > GC_N_MAX) return GC_ERANGE;
  if (!finite_pos(p->sigma_s) || !finite_pos(p->sigma_r)) return GC_EINVAL;
  if (!std::isfinite(p->L) || !std::isfinite(p->U) || !(p->U > p->L)) return GC_EINVAL;
  if (p->op != GC_OP_AUTO && p->op != GC_OP_FIR && p->op != GC_OP_O1 && p->op != GC_OP_DERICHE) return GC_EINVAL;
  if (p->precision != GC_PREC_FP32 && p->precision != GC_PREC_FP64) return GC_EINVAL;
  if (p->op == GC_OP_DERICHE) {
    // recursive mode: fp32 only, all NP <= 8 plane pairs of a column held by one lane
    if (p->precision != GC_PREC_FP32) return GC_EINVAL;
    if ((p->N + 3) / 2 > kDrMaxPairs) return GC_ERANGE;
    if (std::ceil(10.0 * (double)p->sigma_s) > (double)kO1MaxW) return GC_ERANGE;
  }
  if (radius_of(p->sigma_s) > (p->op == GC_OP_FIR || p->precision == GC_PREC_FP64 ? kMaxFirW : kO1MaxW))
    return GC_ERANGE;
  if (p->c) {
    for (int n = 0; n <= p->N; n++)
      if (!std::isfinite(p->c[n])) return GC_EINVAL;
  }
  return GC_OK;
}

// Fill the arithmetic part of KParams (coefficients, taps, centring constants).
gc_status fill_constants(const gc_params* p, KParams& k, std::vector<float2>& taps_host) {
  const double L = p->L, U = p->U;
  const double th = 0.5 * (U - L);
  const double mu = th * th / ((double)p->sigma_r * (double)p->sigma_r);
  std::vector<double> cm(p->N + 1);
  if (p->c) {
    // caller coefficients: c_n mu^n, normalised by the largest magnitude (cancels in P/Q)
    double mx = 0;
    for (int n = 0; n <= p->N; n++) {
      cm[n] = p->c[n] * std::pow(mu, (double)n);
      mx = std::max(mx, std::fabs(cm[n]));
    }
    if (!(mx > 0) || !std::isfinite(mx)) return GC_ERANGE;
    for (auto& v : cm) v /= mx;
  } else {
    gc_status st = coeffs_cached(p->N, p->sigma_r, L, U, nullptr, &cm, nullptr);
    if (st != GC_OK) return st;
  }
  const int planes = ((p->N + 2) + 1) / 2 * 2;
  k.NP = planes / 2;
  for (int n = 0; n < kMaxPlanes; n++) k.chat_d[n] = n <= p->N ? cm[n] : 0.0;
  k.fp64 = p->precision == GC_PREC_FP64;
  k.d_L = L;
  k.d_U = U;
  k.d_tc = 0.5 * (L + U);
  k.d_th = th;
  k.d_inv_th = 1.0 / th;
  k.d_exk = -0.5 * mu;
  for (int q = 0; q < kMaxPairs; q++) {
    const int n0 = 2 * q, n1 = 2 * q + 1;
    k.chat2[q] = make_float2(n0 <= p->N ? (float)cm[n0] : 0.f, n1 <= p->N ? (float)cm[n1] : 0.f);
  }
  k.R = radius_of(p->sigma_s);
  k.sigma_s_host = p->sigma_s;
  std::vector<double> t = taps_of(p->sigma_s, k.R);
  taps_host.resize(t.size());
  for (size_t m = 0; m < t.size(); m++) taps_host[m] = make_float2((float)t[m], (float)t[m]);
  for (int m = 0; m < 2 * kMaxTemplW + 1; m++) k.tap[m] = m < (int)t.size() ? (float)t[m] : 0.f;
  k.L = (float)L;
  k.U = (float)U;
  k.t_c = (float)(0.5 * (L + U));
  k.t_h = (float)th;
  k.inv_th = (float)(1.0 / th);
  k.ex_k = (float)(-0.5 * mu * 1.4426950408889634);
  k.fallback = p->fallback_count;
  for (int i = 0; i < 3; i++) k.ev[i] = reinterpret_cast<cudaEvent_t>(p->events[i]);
  // operator: GC_OP_AUTO = FIR for small radii (fewer instructions), O(1) above
  int op = p->op == GC_OP_AUTO ? (k.R >= kO1AutoMinW ? GC_OP_O1 : GC_OP_FIR) : p->op;
  if (k.fp64) op = GC_OP_FIR;                     // binary64 mode: the exact FIR of eq. (7)
  k.op = op;
  if (op == GC_OP_O1) o1_constants(p->sigma_s, k);
  if (op == GC_OP_DERICHE) deriche_constants(p->sigma_s, k);
  return GC_OK;
}

gc_status cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return GC_OK;
  if (e == cudaErrorMemoryAllocation) return GC_ENOMEM;
  return GC_ECUDA;
}

}  // namespace

// Stream-ordered scratch comes from a libgc-private memory pool per device, never from the
// device's default pool (which PyTorch and other libraries share).  Freed blocks
// stay reserved in the private pool up to its release threshold: unbounded by default, since
// the c5 plane buffer is 14 GiB and re-mapping it on every call costs milliseconds.  The
// environment variable GC_POOL_RELEASE_BYTES bounds it; gc_scratch_trim() hands reserved
// memory back to the driver on demand.
cudaMemPool_t scratch_pool() {
  static std::mutex mu;
  static cudaMemPool_t pools[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lk(mu);
  if (!pools[dev]) {
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t pl = nullptr;
    if (cudaMemPoolCreate(&pl, &props) != cudaSuccess) return nullptr;
    uint64_t thr = UINT64_MAX;
    if (const char* env = std::getenv("GC_POOL_RELEASE_BYTES")) thr = std::strtoull(env, nullptr, 10);
    cudaMemPoolSetAttribute(pl, cudaMemPoolAttrReleaseThreshold, &thr);
    pools[dev] = pl;
  }
  return pools[dev];
}

// GC_BOUNDS_CHECK builds: a per-device counter of out-of-bounds device accesses (gc_device.cuh
// GC_CHK); nullptr in the product library.
unsigned long long* oob_counter() {
#ifdef GC_BOUNDS_CHECK
  static std::mutex mu;
  static unsigned long long* ctr[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lk(mu);
  if (!ctr[dev] && cudaMalloc((void**)&ctr[dev], sizeof(unsigned long long)) == cudaSuccess)
    cudaMemset(ctr[dev], 0, sizeof(unsigned long long));
  return ctr[dev];
#else
  return nullptr;
#endif
}

cudaError_t scratch_alloc(void** ptr, size_t bytes, cudaStream_t s) {
  cudaMemPool_t pl = scratch_pool();
  if (!pl) return cudaErrorInitializationError;
  return cudaMallocFromPoolAsync(ptr, bytes, pl, s);
}

namespace {

// Per-device copy-in / copy-out streams and a second compute stream of gc_filter_host
// (created once, never destroyed).
bool host_streams(cudaStream_t* sin, cudaStream_t* sout, cudaStream_t* sc) {
  static std::mutex mu;
  static cudaStream_t tab[64][3] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return false;
  std::lock_guard<std::mutex> lk(mu);
  for (int i = 0; i < 3; i++)
    if (!tab[dev][i] && cudaStreamCreateWithFlags(&tab[dev][i], cudaStreamNonBlocking) != cudaSuccess) return false;
  *sin = tab[dev][0];
  *sout = tab[dev][1];
  *sc = tab[dev][2];
  return true;
}

// Per-device free list of timing-disabled events for gc_filter_host (creating and destroying
// 2K+2 events per call costs more than a small image's kernels).  Events taken by a call are
// private to it until returned.
struct EventPool {
  std::mutex mu;
  std::vector<cudaEvent_t> free_[64];
  bool take(int n, std::vector<cudaEvent_t>& out) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return false;
    std::lock_guard<std::mutex> lk(mu);
    auto& f = free_[dev];
    out.clear();
    while ((int)out.size() < n && !f.empty()) {
      out.push_back(f.back());
      f.pop_back();
    }
    while ((int)out.size() < n) {
      cudaEvent_t ev = nullptr;
      if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) {
        for (auto e : out) f.push_back(e);
        out.clear();
        return false;
      }
      out.push_back(ev);
    }
    return true;
  }
  void give(const std::vector<cudaEvent_t>& evs) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return;
    std::lock_guard<std::mutex> lk(mu);
    for (auto e : evs) free_[dev].push_back(e);
  }
};
EventPool& event_pool() {
  static EventPool p;
  return p;
}

// Run the pipeline for the window described by k (rows/segments already set).
gc_status run(KParams& k, const std::vector<float2>& taps_host, cudaStream_t s) {
  int dev = 0;
  cudaGetDevice(&dev);
  k.num_sms = 148;
  cudaDeviceGetAttribute(&k.num_sms, cudaDevAttrMultiProcessorCount, dev);
  const int op = k.op;
  const size_t plane_elems = (size_t)k.NP * k.in_rows * k.Wd;
  float2* planes = nullptr;
  float2* taps_dev = nullptr;
  // plane buffer + 256 bytes of task counters at its end
  const size_t elem = k.fp64 ? sizeof(double2) : sizeof(float2);
  // (Deriche mode: a second plane-sized buffer after the counters for the causal partial sums)
  const size_t scratch_elems = op == GC_OP_DERICHE ? plane_elems * k.B : 0;
  // (O(1) mode: the direct lead-in table after the counters)
  const std::vector<float4> lead = op == GC_OP_O1 && !k.fp64 ? o1_lead_table(k.sigma_s_host, k.R) : std::vector<float4>();
  const size_t lead_bytes = lead.size() * sizeof(float4);
  const size_t base_bytes = (plane_elems * k.B * elem + 256 + scratch_elems * elem + 255) / 256 * 256;
  cudaError_t e = scratch_alloc((void**)&planes, base_bytes + lead_bytes, s);
  if (e != cudaSuccess) return cuda_status(e);
  k.counters = reinterpret_cast<unsigned*>(reinterpret_cast<char*>(planes) + plane_elems * k.B * elem);
  k.planes_bytes = base_bytes + lead_bytes;
  k.o1_lead = nullptr;
  if (lead_bytes) {
    float4* lead_dev = reinterpret_cast<float4*>(reinterpret_cast<char*>(planes) + base_bytes);
    e = cudaMemcpyAsync(lead_dev, lead.data(), lead_bytes, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) {
      cudaFreeAsync(planes, s);
      return cuda_status(e);
    }
    k.o1_lead = lead_dev;
  }
  k.oob = oob_counter();
  k.scratch = scratch_elems ? reinterpret_cast<float2*>(reinterpret_cast<char*>(k.counters) + 256) : nullptr;
  if (k.fp64 || (op == GC_OP_FIR && k.R > kMaxTemplW)) {
    // taps for the runtime-radius kernels: (k_m, k_m) fp32 pairs, or k_m in binary64
    std::vector<double> td;
    const void* src = taps_host.data();
    size_t bytes = taps_host.size() * sizeof(float2);
    if (k.fp64) {
      td = taps_of(k.sigma_s_host, k.R);
      src = td.data();
      bytes = td.size() * sizeof(double);
    }
    e = scratch_alloc((void**)&taps_dev, bytes, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(taps_dev, src, bytes, cudaMemcpyHostToDevice, s);
    // (pageable source: cudaMemcpyAsync returns once the bytes are staged, td may then go)
    if (e != cudaSuccess) {
      cudaFreeAsync(planes, s);
      if (taps_dev) cudaFreeAsync(taps_dev, s);
      return cuda_status(e);
    }
  }
  k.planes = planes;
  k.planes_img_stride = (long long)plane_elems;
  k.taps_g = taps_dev;
  k.taps_d = reinterpret_cast<const double*>(taps_dev);
  e = k.fp64                ? launch_fp64_two_pass(k, s)
      : op == GC_OP_O1      ? launch_o1_two_pass(k, s)
      : op == GC_OP_DERICHE ? launch_deriche_two_pass(k, s)
                            : launch_fir_two_pass(k, s);
  cudaError_t e2 = cudaFreeAsync(planes, s);
  if (taps_dev) cudaFreeAsync(taps_dev, s);
  if (e != cudaSuccess) return cuda_status(e);
  return cuda_status(e2);
}

}  // namespace
}  // namespace gc

using namespace gc;

extern "C" {

const char* gc_status_string(gc_status s) {
  switch (s) {
    case GC_OK: return "GC_OK";
    case GC_EINVAL: return "GC_EINVAL: invalid argument";
    case GC_ERANGE: return "GC_ERANGE: parameter outside the supported range";
    case GC_ECUDA: return "GC_ECUDA: CUDA error";
    case GC_ENOMEM: return "GC_ENOMEM: device allocation failed";
    case GC_ENCCL: return "GC_ENCCL: NCCL error";
    case GC_ETIMEOUT: return "GC_ETIMEOUT: collective did not complete in time (communicator aborted)";
  }
  return "GC_?: unknown status";
}

const char* gc_version(void) {
#ifdef GC_BOUNDS_CHECK
  return "gc 0.2.0 sm_100a +bounds-check";
#else
  return "gc 0.2.0 sm_100a";
#endif
}

gc_status gc_debug_oob_count(unsigned long long* count) {
  if (!count) return GC_EINVAL;
  unsigned long long* c = oob_counter();
  if (!c) return GC_ERANGE;                       // not a GC_BOUNDS_CHECK build
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaMemcpy(count, c, sizeof(*count), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemset(c, 0, sizeof(*count));
  return cuda_status(e);
}

gc_status gc_debug_oob_selftest(void) {
  unsigned long long* c = oob_counter();
  if (!c) return GC_ERANGE;                       // not a GC_BOUNDS_CHECK build
  KParams k;
  std::memset(&k, 0, sizeof(k));
  float2* buf = nullptr;
  cudaError_t e = cudaMalloc((void**)&buf, 4096);
  if (e != cudaSuccess) return cuda_status(e);
  k.planes = buf;
  k.planes_bytes = 4096;
  k.oob = c;
  e = launch_oob_selftest(k, nullptr);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  cudaFree(buf);
  return cuda_status(e);
}

gc_status gc_scratch_trim(size_t keep_bytes) {
  cudaMemPool_t pl = scratch_pool();
  if (!pl) return GC_ECUDA;
  return cuda_status(cudaMemPoolTrimTo(pl, keep_bytes));
}

void gc_params_init(gc_params* p, int N, float sigma_s, float sigma_r) {
  if (!p) return;
  std::memset(p, 0, sizeof(*p));
  p->N = N;
  p->sigma_s = sigma_s;
  p->sigma_r = sigma_r;
  p->L = 0.f;
  p->U = 255.f;
  p->c = nullptr;
  p->op = GC_OP_AUTO;
  p->fallback_count = nullptr;
}

gc_status gc_filter_window(const float* const seg[3], const int seg_row0[3], const int seg_rows[3],
                           int H_global, int W, int out_row0, int out_rows, const gc_params* p,
                           float* out, void* stream) {
  gc_status st = validate_params(p);
  if (st != GC_OK) return st;
  if (!seg || !seg_row0 || !seg_rows || !out) return GC_EINVAL;
  if (H_global < 1 || W < 1 || out_rows < 1 || out_row0 < 0 || out_row0 + out_rows > H_global)
    return GC_EINVAL;
  KParams k;
  std::memset(&k, 0, sizeof(k));
  int nseg = 0;
  for (int i = 0; i < 3; i++) {
    if (seg_rows[i] == 0) { k.seg[i] = Seg{seg[i], -1, 0}; continue; }
    if (seg_rows[i] < 0 || !seg[i] || seg_row0[i] < 0 || seg_row0[i] + seg_rows[i] > H_global) return GC_EINVAL;
    if (overlap(seg[i], (size_t)seg_rows[i] * W * 4, out, (size_t)out_rows * W * 4)) return GC_EINVAL;
    k.seg[i] = Seg{seg[i], seg_row0[i], seg_rows[i]};
    nseg++;
  }
  if (nseg == 0) return GC_EINVAL;
  const int R = halo_of(p);
  // rows the window needs (after symmetric extension) must all be in some segment
  int lo = H_global, hi = -1;
  auto mir = [&](int q) {
    if (H_global == 1) return 0;
    const int per = 2 * H_global - 2;
    q = q < 0 ? -q : q;
    q %= per;
    return q < H_global ? q : per - q;
  };
  for (int y = out_row0 - R; y <= out_row0 + out_rows - 1 + R; y++) {
    const int q = mir(y);
    bool found = false;
    for (int i = 0; i < 3; i++)
      if (k.seg[i].rows > 0 && q >= k.seg[i].row0 && q < k.seg[i].row0 + k.seg[i].rows) found = true;
    if (!found) return GC_EINVAL;
    lo = std::min(lo, q);
    hi = std::max(hi, q);
  }
  std::vector<float2> taps_host;
  st = fill_constants(p, k, taps_host);
  if (st != GC_OK) return st;
  k.H = H_global;
  k.Wd = W;
  k.B = 1;
  k.in_row0 = lo;
  k.in_rows = hi - lo + 1;
  k.out_row0 = out_row0;
  k.out_rows = out_rows;
  k.seg_img_stride = 0;
  k.out = out;
  k.out_img_stride = (long long)out_rows * W;
  return run(k, taps_host, reinterpret_cast<cudaStream_t>(stream));
}

gc_status gc_filter(const float* imgs, int B, int H, int W, const gc_params* p, float* outs, void* stream) {
  gc_status st = validate_params(p);
  if (st != GC_OK) return st;
  if (!imgs || !outs || B < 1 || H < 1 || W < 1) return GC_EINVAL;
  const size_t bytes = (size_t)B * H * W * sizeof(float);
  if (overlap(imgs, bytes, outs, bytes)) return GC_EINVAL;
  KParams k;
  std::memset(&k, 0, sizeof(k));
  std::vector<float2> taps_host;
  st = fill_constants(p, k, taps_host);
  if (st != GC_OK) return st;
  k.H = H;
  k.Wd = W;
  k.B = B;
  k.in_row0 = 0;
  k.in_rows = H;
  k.out_row0 = 0;
  k.out_rows = H;
  k.seg[0] = Seg{imgs, 0, H};
  k.seg[1] = Seg{imgs, -1, 0};
  k.seg[2] = Seg{imgs, -1, 0};
  k.seg_img_stride = (long long)H * W;
  k.out = outs;
  k.out_img_stride = (long long)H * W;
  return run(k, taps_host, reinterpret_cast<cudaStream_t>(stream));
}

gc_status gc_filter_kernels(int B, int H, int W, const gc_params* p, int* n_kernels) {
  gc_status st = validate_params(p);
  if (st != GC_OK) return st;
  if (!n_kernels || B < 1 || H < 1 || W < 1) return GC_EINVAL;
  KParams k;
  std::memset(&k, 0, sizeof(k));
  std::vector<float2> taps_host;
  st = fill_constants(p, k, taps_host);
  if (st != GC_OK) return st;
  k.H = H;
  k.Wd = W;
  k.B = B;
  k.in_rows = k.out_rows = H;
  *n_kernels = fused_fir_applies(k) ? 1 : 2;
  return GC_OK;
}

gc_status gc_gaussian(const float* imgs, int B, int H, int W, float sigma_s, int op, float* outs, void* stream) {
  gc_params p;
  gc_params_init(&p, 0, sigma_s, 1000.f);   // N = 0, one plane pair (f, 0); sigma_r unused
  p.op = op;
  gc_status st = validate_params(&p);
  if (st != GC_OK) return st;
  if (!imgs || !outs || B < 1 || H < 1 || W < 1) return GC_EINVAL;
  const size_t bytes = (size_t)B * H * W * sizeof(float);
  if (overlap(imgs, bytes, outs, bytes)) return GC_EINVAL;
  KParams k;
  std::memset(&k, 0, sizeof(k));
  std::vector<float2> taps_host;
  st = fill_constants(&p, k, taps_host);
  if (st != GC_OK) return st;
  k.raw = 1;
  k.H = H;
  k.Wd = W;
  k.B = B;
  k.in_row0 = 0;
  k.in_rows = H;
  k.out_row0 = 0;
  k.out_rows = H;
  k.seg[0] = Seg{imgs, 0, H};
  k.seg[1] = Seg{imgs, -1, 0};
  k.seg[2] = Seg{imgs, -1, 0};
  k.seg_img_stride = (long long)H * W;
  k.out = outs;
  k.out_img_stride = (long long)H * W;
  return run(k, taps_host, reinterpret_cast<cudaStream_t>(stream));
}

gc_status gc_bilateral_direct(const float* imgs, int B, int H, int W, float sigma_s, float sigma_r, float* outs,
                              void* stream) {
  if (!imgs || !outs || B < 1 || H < 1 || W < 1) return GC_EINVAL;
  if (!finite_pos(sigma_s) || !finite_pos(sigma_r)) return GC_EINVAL;
  const size_t bytes = (size_t)B * H * W * sizeof(float);
  if (overlap(imgs, bytes, outs, bytes)) return GC_EINVAL;
  const int R = radius_of(sigma_s);
  if (R > kMaxFirW) return GC_ERANGE;
  return cuda_status(launch_direct(imgs, B, H, W, R, sigma_s, sigma_r, outs, reinterpret_cast<cudaStream_t>(stream)));
}

gc_status gc_operator_taps(float sigma_s, int op, double* taps_out, int* W_out) {
  if (!std::isfinite(sigma_s) || !(sigma_s > 0)) return GC_EINVAL;
  if (op != GC_OP_AUTO && op != GC_OP_FIR && op != GC_OP_O1) return GC_EINVAL;
  const int R = radius_of(sigma_s);
  if (R > (op == GC_OP_FIR ? kMaxFirW : kO1MaxW)) return GC_ERANGE;
  if (op == GC_OP_AUTO) op = R >= kO1AutoMinW ? GC_OP_O1 : GC_OP_FIR;
  if (W_out) *W_out = R;
  if (!taps_out) return GC_OK;
  if (op == GC_OP_FIR) {
    const std::vector<double> t = taps_of(sigma_s, R);
    std::copy(t.begin(), t.end(), taps_out);
  } else {
    const O1Fit f = o1_fit_cached(sigma_s);
    for (int m = -R; m <= R; m++) {
      double v = 0;
      for (int q = 0; q < kO1K; q++) v += f.alpha[q] * std::cos(f.omega[q] * m);
      taps_out[m + R] = v;
    }
  }
  return GC_OK;
}

gc_status gc_bilateral(const float* img, int H, int W, float sigma_s, float sigma_r, int N, float* out,
                       void* stream) {
  gc_params p;
  gc_params_init(&p, N, sigma_s, sigma_r);
  return gc_filter(img, 1, H, W, &p, out, stream);
}

gc_status gc_bilateral_batch(const float* imgs, int B, int H, int W, float sigma_s, float sigma_r, int N,
                             float* outs, void* stream) {
  gc_params p;
  gc_params_init(&p, N, sigma_s, sigma_r);
  return gc_filter(imgs, B, H, W, &p, outs, stream);
}

gc_status gc_bilateral_c(const float* img, int H, int W, float sigma_s, float sigma_r, int N, const double* c,
                         float* out, void* stream) {
  if (!c) return GC_EINVAL;
  gc_params p;
  gc_params_init(&p, N, sigma_s, sigma_r);
  p.c = c;
  return gc_filter(img, 1, H, W, &p, out, stream);
}

gc_status gc_filter_host(const float* imgs_host, int B, int H, int W, const gc_params* p, float* outs_host,
                         void* stream) {
  gc_status st = validate_params(p);
  if (st != GC_OK) return st;
  if (!imgs_host || !outs_host || B < 1 || H < 1 || W < 1) return GC_EINVAL;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  // GC_HOST_TRACE=1: print the pipeline's device timeline and host enqueue time (development)
  static const bool trace = std::getenv("GC_HOST_TRACE") != nullptr;
  const auto t_host0 = std::chrono::steady_clock::now();
  const size_t bytes = (size_t)B * H * W * sizeof(float);
  float *din = nullptr, *dout = nullptr;
  cudaError_t e = scratch_alloc((void**)&din, bytes, s);
  if (e != cudaSuccess) return cuda_status(e);
  e = scratch_alloc((void**)&dout, bytes, s);
  if (e != cudaSuccess) { cudaFreeAsync(din, s); return cuda_status(e); }
  // Pipeline: the input is copied in K chunks on a copy-in stream, each chunk is filtered on
  // `s` as soon as the rows it reads have arrived, and copied back on a copy-out stream, so the
  // two PCIe directions and the kernels overlap.  Chunks are images (B > 1) or row bands of one
  // image (B = 1, gc_filter_window over the whole device image; halo rows come from the
  // neighbouring chunks' copies).  Results are identical to gc_filter up to the O(1)
  // operator's segment-dependent rounding (FIR: bit-identical).
  const int R = halo_of(p);
  // chunks of >= 2 MB, at most 8 for batches, and for row bands >= max(8 R, 64) rows
  // (measured on B200, tools/host_timing1.py, profiles/r01_e2e_host_chunks.txt: c2 device
  // timeline 171 us with 2 chunks vs 193 with 4 and 207 with 1 (GC_HOST_TRACE; H2D and D2H
  // barely overlap on this PCIe link, so 8 MB of copies take >= 155 us); c5 16 chunks 25.7 ms
  // vs 8: 29.5, 32: 26.8; c1 1 chunk 76 us vs 2: 104; c4 x32 8 chunks 3.79 ms vs 16: 3.92)
  int K = (int)std::max<size_t>(1, std::min<size_t>(16, bytes / (2u << 20)));
  if (B > 1) K = std::min(std::min(K, 8), B);
  else K = std::max(1, std::min(K, H / std::max(64, 8 * R)));
  if (const char* env = std::getenv("GC_HOST_CHUNKS")) K = std::max(1, std::min(atoi(env), B > 1 ? B : H));
  cudaStream_t sin = nullptr, sout = nullptr, sc = nullptr;
  std::vector<cudaEvent_t> evs, tr;
  const bool ok = host_streams(&sin, &sout, &sc) && event_pool().take(2 * K + 3, evs);
  cudaEvent_t* ev_in = ok ? evs.data() : nullptr;
  cudaEvent_t* ev_comp = ok ? evs.data() + K : nullptr;
  cudaEvent_t ev_start = ok ? evs[2 * K] : nullptr, ev_done = ok ? evs[2 * K + 1] : nullptr;
  cudaEvent_t ev_c2 = ok ? evs[2 * K + 2] : nullptr;
  if (!ok) {
    st = GC_ECUDA;
  } else {
    // output chunk k = [c0[k], c0[k+1]) images (B > 1) or rows (B = 1).  For row bands the
    // input chunks are shifted down by the halo, h[k] = c0[k] + R, so that band k reads only
    // input chunks 0..k and starts as soon as chunk k has arrived.
    const int n = B > 1 ? B : H;
    std::vector<int> c0(K + 1), h(K + 1);
    for (int k = 0; k <= K; k++) c0[k] = (int)((long long)n * k / K);
    for (int k = 0; k <= K; k++) h[k] = (B > 1 || k == 0 || k == K) ? c0[k] : std::min(n, c0[k] + R);
    const size_t unit = B > 1 ? (size_t)H * W : (size_t)W;     // floats per image / per row
    cudaEventRecord(ev_start, s);                                // device buffers allocated
    cudaStreamWaitEvent(sin, ev_start, 0);
    cudaStreamWaitEvent(sc, ev_start, 0);
    if (trace) {
      tr.resize(3 * K + 1);
      for (auto& ev : tr) cudaEventCreate(&ev);
      cudaEventRecord(tr[0], s);
    }
    for (int k = 0; k < K && e == cudaSuccess; k++) {
      const size_t off = (size_t)h[k] * unit, cnt = (size_t)(h[k + 1] - h[k]) * unit;
      if (cnt) e = cudaMemcpyAsync(din + off, imgs_host + off, cnt * 4, cudaMemcpyHostToDevice, sin);
      if (e == cudaSuccess) e = cudaEventRecord(ev_in[k], sin);
      if (trace) cudaEventRecord(tr[1 + k], sin);
    }
    // row bands alternate between two compute streams, so a band's kernels overlap the
    // previous band's tail (a band of one image does not fill the GPU on its own; image
    // chunks of a batch do, and stay on `s`)
    for (int k = 0; k < K && e == cudaSuccess && st == GC_OK; k++) {
      cudaStream_t sk = (B == 1 && (k & 1)) ? sc : s;
      cudaStreamWaitEvent(sk, ev_in[k], 0);                     // input chunks 0..k have arrived
      if (B > 1) {
        st = gc_filter(din + (size_t)c0[k] * unit, c0[k + 1] - c0[k], H, W, p, dout + (size_t)c0[k] * unit, sk);
      } else {
        const float* seg[3] = {din, din, din};
        const int seg_row0[3] = {0, -1, -1};
        const int seg_rows[3] = {H, 0, 0};
        st = gc_filter_window(seg, seg_row0, seg_rows, H, W, c0[k], c0[k + 1] - c0[k], p,
                              dout + (size_t)c0[k] * unit, sk);
      }
      if (st == GC_OK) e = cudaEventRecord(ev_comp[k], sk);
      if (trace) cudaEventRecord(tr[1 + K + k], sk);
    }
    for (int k = 0; k < K && e == cudaSuccess && st == GC_OK; k++) {
      const size_t off = (size_t)c0[k] * unit, cnt = (size_t)(c0[k + 1] - c0[k]) * unit;
      cudaStreamWaitEvent(sout, ev_comp[k], 0);
      e = cudaMemcpyAsync(outs_host + off, dout + off, cnt * 4, cudaMemcpyDeviceToHost, sout);
      if (trace) cudaEventRecord(tr[1 + 2 * K + k], sout);
    }
    cudaEventRecord(ev_done, sout);
    cudaEventRecord(ev_start, sin);
    cudaEventRecord(ev_c2, sc);
    cudaStreamWaitEvent(s, ev_done, 0);                          // buffers free only after all
    cudaStreamWaitEvent(s, ev_start, 0);                         // copies and both compute
    cudaStreamWaitEvent(s, ev_c2, 0);                            // streams
  }
  cudaFreeAsync(din, s);
  cudaFreeAsync(dout, s);
  const auto t_host1 = std::chrono::steady_clock::now();
  cudaError_t es = cudaStreamSynchronize(s);
  if (ok) event_pool().give(evs);
  if (trace && !tr.empty()) {
    const auto t_host2 = std::chrono::steady_clock::now();
    auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
    std::fprintf(stderr, "gc_filter_host K=%d: host enqueue %.1f us, sync wait %.1f us | device (us from start):", K,
                 us(t_host0, t_host1), us(t_host1, t_host2));
    const char* what[3] = {"h2d", "comp", "d2h"};
    for (int w = 0; w < 3; w++) {
      std::fprintf(stderr, " %s", what[w]);
      for (int k = 0; k < K; k++) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, tr[0], tr[1 + w * K + k]);
        std::fprintf(stderr, " %.1f", 1e3f * ms);
      }
    }
    std::fprintf(stderr, "\n");
    for (auto ev : tr) cudaEventDestroy(ev);
  }
  if (st != GC_OK) return st;
  if (e != cudaSuccess) return cuda_status(e);
  return cuda_status(es);
}

}  // extern "C"
