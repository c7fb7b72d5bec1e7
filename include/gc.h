/*
 * gc.h — C ABI of libgc: the Gauss–Chebyshev fast bilateral filter (GCF) hot path
 * on NVIDIA B200 (sm_100a).
 *
 * Paper: S. Ghosh, K. N. Chaudhury, "Fast and High-Quality Bilateral Filtering Using
 * Gauss-Chebyshev Approximation", arXiv 1605.02178 (IEEE SPCOM 2016).  Citations below
 * are `P:<line>` = line of /root/reference/PAPER.md (section / equation in brackets).
 *
 * Problem statement (what every entry point computes):
 *   f : I -> R, I a finite H x W rectangle of Z^2, one fp32 grayscale image, row-major,
 *   pitch W; extended outside I by whole-sample symmetry (P:36 [Sec. I]; R5).
 *   Spatial kernel g_{sigma_s}(j) = exp(-|j|^2 / 2 sigma_s^2) on Omega = [-W_s, W_s]^2,
 *   W_s = ceil(3 sigma_s) (P:39, P:48 [Sec. I]; R4).  Range kernel g_{sigma_r}(t) =
 *   exp(-t^2 / 2 sigma_r^2).  Intensity range [L, U], default [0, 255].
 *   Output: the GCF approximation of the bilateral filter, eq. (10) (P:108-111 [Sec. II]),
 *   computed by the pipeline of P:235-240 [Sec. III-B]:
 *     g = clamp(f, L, U) - t_c, t_c = (L+U)/2                     eq. (17)
 *     c_n = Chebyshev coefficients of exp on [-mu, mu]            eq. (19)
 *     F_n = exp(-g^2/2sr^2) (g/sr)^n, n = 0..N+1;  G_n = (g/sr)^n eq. (6)
 *     Fbar_n = sum_{j in Omega} g_{sigma_s}(j) F_n(i-j)           eq. (7)
 *     P = sr sum_n c_n G_n Fbar_{n+1},  Q = sum_n c_n G_n Fbar_n  eqs. (8),(9) P:97-106
 *     out = P/Q + t_c   where Q > 0 and finite, else out = clamp(f)(i)  (R8)
 *
 * Conventions for all entry points
 *   - Status codes, never exceptions; nothing is printed.
 *   - Device entry points are asynchronous on `stream` (a cudaStream_t passed as void*;
 *     NULL = legacy default stream).  They return after enqueue.  Argument errors are
 *     detected before anything is enqueued.  Kernel execution errors surface at the
 *     caller's next synchronisation with the stream.
 *   - Image memory is owned by the caller.  The library owns bounded, mutex-guarded constant
 *     caches and stream-ordered scratch (cudaMallocFromPoolAsync / cudaFreeAsync on `stream`,
 *     from a libgc-private memory pool per device; see gc_scratch_trim).
 *   - All entry points are re-entrant and thread-safe.
 *   - `out` must not alias the input.
 *   - NaN/Inf inputs give unspecified output values (no fault).
 */
#ifndef GC_H_
#define GC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  GC_OK = 0,
  GC_EINVAL = 1,  /* bad argument (sizes, sigmas, N, null or aliased pointers)        */
  GC_ERANGE = 2,  /* N > GC_N_MAX, or mu beyond the coefficient precision limit        */
  GC_ECUDA = 3,   /* a CUDA call or kernel launch failed                               */
  GC_ENOMEM = 4,  /* device scratch allocation failed                                  */
  GC_ENCCL = 5,   /* an NCCL call failed, or a peer reported an asynchronous error     */
  GC_ETIMEOUT = 6 /* gc_comm_wait: the exchange did not complete in time (comm aborted) */
} gc_status;

#define GC_N_MAX 64          /* maximum polynomial degree N                           */
#define GC_MU_MAX 4096.0     /* maximum mu = (U-L)^2 / (4 sigma_r^2) for gc_coeffs    */

/* Spatial operator used for eq. (7).  FIR and O1 compute the truncated sum over Omega
   exactly as eq. (7) writes it (R3); they differ only in cost and rounding.
   DERICHE replaces it by the recursive filter the paper cites for its O(1) claim. */
typedef enum {
  GC_OP_AUTO = 0,  /* library choice by W_s: FIR for W_s <= 24, O1 above  */
  GC_OP_FIR = 1,   /* direct separable FIR, 2(2W_s+1) FMA per plane-pixel; W_s <= 1024   */
  GC_OP_O1 = 2,    /* exact-window O(1) recursion: the truncated window of eq. (7) with
                      the taps replaced by a 5-term cosine fit with optimised frequencies
                      (max error ~5e-8 of the peak tap); 24 packed FP32x2 ops per plane-pixel
                      pair and pass,
                      independent of sigma_s; W_s <= 4096                                  */
  GC_OP_DERICHE = 3 /* NOT eq. (7): the untruncated 4th-order recursive Gaussian of
                      [Deriche1993] that P:50 / P:112 cite for the O(1) claim (SURVEY §8(f)
                      NEXT-1): causal + anticausal recursions on each line padded with
                      ceil(10 sigma_s) mirrored samples, zero initial state.  Opt-in only
                      (GC_OP_AUTO never picks it); N <= 14; fp32 only; windows and bands
                      need K = ceil(10 sigma_s) halo rows instead of W_s.  Moves the GCF by
                      ~0.2-0.35 grey levels against eq. (7)                */
} gc_operator;

/* Human-readable name of a status code (static storage). */
const char* gc_status_string(gc_status s);

/* Library version string, e.g. "gc 0.2.0 sm_100a". */
const char* gc_version(void);

/*
 * gc_coeffs — host only, pure, thread-safe.
 * c_out[0..N] = eq. (19) coefficients c_n of the degree-N Chebyshev
 * interpolant of exp on [-mu, mu] (eq. 16 with the nodes rescaled),
 * mu = (U-L)^2 / (4 sigma_r^2), computed in the library's own multiprecision
 * arithmetic (>= mu/ln10 + 40 significant digits; R2) and rounded once to
 * binary64.  mu_out (may be NULL) receives mu rounded to binary64.
 * Errors: GC_EINVAL if c_out is NULL, N < 0, !(sigma_r > 0), !(U > L) or any argument
 * is non-finite; GC_ERANGE if N > GC_N_MAX or mu > GC_MU_MAX.
 */
gc_status gc_coeffs(int N, double sigma_r, double L, double U, double* c_out, double* mu_out);

/*
 * gc_bilateral — one image on the device.
 * img, out: device pointers to H*W fp32, row-major, pitch W.  L = 0, U = 255.
 * Errors: GC_EINVAL (H < 1, W < 1, !(sigma_s > 0), !(sigma_r > 0), N < 0, null or
 * overlapping img/out, non-finite sigmas), GC_ERANGE (N > GC_N_MAX, mu > GC_MU_MAX),
 * GC_ECUDA (launch failure).
 */
gc_status gc_bilateral(const float* img, int H, int W, float sigma_s, float sigma_r, int N,
                       float* out, void* stream);

/*
 * gc_bilateral_batch — B images, contiguous [B][H][W] fp32 on the device, same
 * parameters for all; outs has the same layout.  B >= 1.  Errors as gc_bilateral.
 */
gc_status gc_bilateral_batch(const float* imgs, int B, int H, int W, float sigma_s,
                             float sigma_r, int N, float* outs, void* stream);

/*
 * gc_bilateral_c — as gc_bilateral with caller-supplied coefficients c[0..N] (host
 * pointer, binary64) in place of eq. (19): e.g. c_n = 1/n! gives the Gauss-polynomial
 * filter (GPF) of [Chaudhury2015].  GC_EINVAL if c is NULL or non-finite.
 */
gc_status gc_bilateral_c(const float* img, int H, int W, float sigma_s, float sigma_r, int N,
                         const double* c, float* out, void* stream);

/* Full-control entry point used by the three calls above. */
typedef struct gc_params {
  int N;                              /* degree, 0 <= N <= GC_N_MAX                      */
  float sigma_s;                      /* spatial sigma (pixels) > 0                      */
  float sigma_r;                      /* range sigma (intensity units) > 0               */
  float L, U;                         /* intensity range, U > L                   */
  const double* c;                    /* NULL: eq. (19) coefficients; else host c[0..N]  */
  int op;                             /* gc_operator                                     */
  unsigned long long* fallback_count; /* NULL or device counter; += guarded pixels (R8)  */
  void* events[3];                    /* NULL or cudaEvent_t recorded on `stream` before
                                         the row pass, between the passes and after the
                                         column pass (per-kernel timing for bench.py)      */
  int precision;                      /* GC_PREC_FP32 (default) or GC_PREC_FP64: planes,
                                         eq. (7) and eqs. (8)-(10) in binary64 (FIR
                                         operator, W_s <= 1024; input/output stay fp32)    */
} gc_params;

#define GC_PREC_FP32 0
#define GC_PREC_FP64 1

/* Fill p with the defaults: L=0, U=255, c=NULL, op=GC_OP_AUTO, fallback_count=NULL,
   events={NULL}, precision=GC_PREC_FP32. */
void gc_params_init(gc_params* p, int N, float sigma_s, float sigma_r);

/* B images [B][H][W] on the device (B >= 1). Errors as gc_bilateral. */
gc_status gc_filter(const float* imgs, int B, int H, int W, const gc_params* p, float* outs,
                    void* stream);

/*
 * gc_filter_kernels — the number of kernels gc_filter(imgs, B, H, W, p, ...) launches on its
 * stream, without launching anything (host only): 1 when the call takes the small-image fused
 * FIR kernel (operator FIR, W_s <= 24, B*H*W at most GC_FUSED_MAX_PX output pixels: both passes
 * of eq. (7) P:92-96 and eqs. (8)-(10) in one launch, csrc/gc_fused.cu), else 2 (the two passes;
 * the O(1) path also zeroes a 4-byte task counter with a memset node).  With p->events set, a
 * fused call records events[0] before and events[1], events[2] after its one kernel.
 * Errors: GC_EINVAL / GC_ERANGE as gc_filter's parameter checks, GC_EINVAL for a null n_kernels.
 */
#define GC_FUSED_MAX_PX (1 << 18)
gc_status gc_filter_kernels(int B, int H, int W, const gc_params* p, int* n_kernels);

/*
 * gc_filter_host — end-to-end call on HOST buffers (pinned memory recommended):
 * copies imgs (B*H*W fp32) host->device, filters, copies the result device->host into
 * outs, all on `stream`, and returns after synchronising that stream (so outs is
 * valid on return).  Device buffers are stream-ordered scratch owned by the library.
 * Errors as gc_filter, plus GC_ENOMEM.
 */
gc_status gc_filter_host(const float* imgs_host, int B, int H, int W, const gc_params* p,
                         float* outs_host, void* stream);

/*
 * gc_gaussian — eq. (7) alone: the separable spatial Gaussian over the truncated
 * window Omega = [-W_s, W_s]^2 with whole-sample symmetric extension, applied to B images
 * [B][H][W] fp32 on the device (no centring, no clamping), with operator `op`.  This is the
 * N+2-fold inner step of the GCF exposed on its own (operator tests, impulse responses).
 * Errors: GC_EINVAL (sizes, sigma_s, op, null or overlapping pointers), GC_ERANGE (W_s above
 * the operator's limit), GC_ECUDA.
 */
gc_status gc_gaussian(const float* imgs, int B, int H, int W, float sigma_s, int op, float* outs,
                      void* stream);

/*
 * gc_bilateral_direct — the direct bilateral filter of eq. (1), the O(sigma_s^2)
 * filter the GCF approximates: B images [B][H][W] fp32 on the device, Omega = [-W_s, W_s]^2,
 * W_s = ceil(3 sigma_s), whole-sample symmetric extension, Gaussian spatial and
 * range kernels, fp32 arithmetic (one exp per tap; cost (2 W_s + 1)^2 per pixel).  A reference
 * for full-image MSE / PSNR of the fast filter; not on the GCF hot path.
 * Errors: GC_EINVAL (sizes, sigmas, null or overlapping pointers), GC_ERANGE (W_s > 1024),
 * GC_ECUDA.
 */
gc_status gc_bilateral_direct(const float* imgs, int B, int H, int W, float sigma_s, float sigma_r,
                              float* outs, void* stream);

/*
 * gc_operator_taps — host only, pure: the 1-D impulse response k[m], m = -W_s..W_s, that
 * operator `op` applies along each axis at sigma_s (GC_OP_FIR: the normalised sampled taps of
 * eq. 7; GC_OP_O1: the cosine expansion the O(1) kernels evaluate; GC_OP_AUTO: whichever
 * gc_filter would pick).  taps_out: 2 W_s + 1 doubles (may be NULL to query W_s only);
 * W_out (may be NULL) receives W_s.  Errors: GC_EINVAL, GC_ERANGE.
 */
gc_status gc_operator_taps(float sigma_s, int op, double* taps_out, int* W_out);

/*
 * Row-band API (multi-GPU domain decomposition, one process per GPU).
 *
 * The global image has H_global rows of width W.  Rank r of `world` owns the
 * contiguous rows [row0, row0 + H_band) (ranks ordered by row0; rank r-1 owns the rows
 * above).  Eq. (7) at row y reads rows y-W_s .. y+W_s (Omega) and the auxiliary
 * planes of eq. (6) are pointwise in f, so a band needs only `halo` rows of f from
 * each neighbour: halo = W_s = ceil(3 sigma_s) for GC_OP_AUTO / FIR / O1, ceil(10 sigma_s)
 * for GC_OP_DERICHE.  Symmetric extension applies only at global rows 0 and
 * H_global-1.  Every band must have H_band > halo rows (halos come from the adjacent rank
 * only; GC_EINVAL otherwise).
 *
 * gc_band_plan — host only, pure: the halo rows rank `rank` needs, in global row
 * indices, for operator `op`: top = [top0, top0+top_rows) from rank-1, bottom =
 * [bot0, bot0+bot_rows) from rank+1 (0 rows at the global top / bottom, where eq. 7's
 * symmetric extension is applied locally).  band_rows[k] = rows of rank k (sum H_global).
 * Identical on every rank.  Bands passed to gc_filter_band must come from this plan: it
 * rejects any band that is too small for `op` on EVERY rank alike, so an invalid plan
 * fails before any rank enters the exchange.
 */
gc_status gc_band_plan(int H_global, int rank, int world, const int* band_rows, float sigma_s,
                       int op, int* row0, int* top0, int* top_rows, int* bot0, int* bot_rows);

/* One halo transfer of a band with one neighbour (gc_band_exchange_plan). */
typedef struct gc_band_xfer {
  int peer;             /* neighbour rank, or -1 (global edge: no transfer)                 */
  size_t send_offset;   /* first float of this band sent to `peer` (a row offset times W)   */
  size_t count;         /* floats sent to and received from `peer` (halo rows times W)      */
  int recv_row0;        /* global row of the first received row                             */
} gc_band_xfer;

/*
 * gc_band_exchange_plan — host only, pure: exactly what gc_filter_band exchanges and
 * filters.  xfer[0] = with rank-1 (send my first `halo` rows, receive the `halo` rows above
 * me), xfer[1] = with rank+1 (send my last `halo` rows, receive the rows below me);
 * seg_row0/seg_rows = the three input segments (top halo, own band, bottom halo) then
 * given to gc_filter_window.  Testable without a GPU (tests/test_dist_gloo.py runs this
 * plan over gloo).  GC_EINVAL on inconsistent arguments (rank 0 must start at row 0, the
 * last rank must end at H_global, H_band > halo when world > 1).
 */
gc_status gc_band_exchange_plan(int H_band, int W, int H_global, int row0, int rank, int world,
                                float sigma_s, int op, gc_band_xfer xfer[2], int seg_row0[3],
                                int seg_rows[3]);

/* NCCL communicator owned by the library.  gc_comm_unique_id fills 128 bytes on one
   rank; the caller broadcasts them (e.g. torch.distributed); every rank then calls
   gc_comm_init.  GC_ENCCL on failure.  The CUDA device must be set by the caller.
   `comm` arguments below are that handle (an ncclComm_t passed as void*). */
gc_status gc_comm_unique_id(unsigned char id[128]);
gc_status gc_comm_init(int rank, int world, const unsigned char id[128], void** comm_out);
gc_status gc_comm_destroy(void* comm);

/*
 * gc_comm_wait — host-blocking watchdog for the band exchange: waits until all work on
 * `stream` has completed (GC_OK), polling ncclCommGetAsyncError every ~50 us.  An
 * asynchronous NCCL error aborts the communicator (ncclCommAbort) and returns GC_ENCCL; no
 * completion within timeout_ms (e.g. a peer failed before posting its half of the
 * exchange) aborts it and returns GC_ETIMEOUT.  After an abort the communicator must be
 * destroyed and re-created.  GC_ECUDA if the stream reports a CUDA error.
 */
gc_status gc_comm_wait(void* comm, void* stream, double timeout_ms);

/*
 * gc_bilateral_band — SURVEY §8(b)'s band entry point: this rank's band of the GCF of the
 * global image, with (sigma_s, sigma_r, N) and the defaults of gc_params_init (L = 0,
 * U = 255, eq. 19 coefficients, GC_OP_AUTO).  band / out: device pointers to H_band*W fp32
 * (rows [row0, row0+H_band)).  comm: the ncclComm_t from gc_comm_init (as void*; §8(b)
 * writes it as ncclComm_t).  Collective over comm: exchanges the halo rows of f (not of the
 * N+2 planes: they are pointwise in f, so f is the smallest thing to send) with ranks r-1
 * and r+1 by grouped ncclSend/ncclRecv on `stream` (the plan of gc_band_exchange_plan), then
 * filters; symmetric extension only at global rows 0 and H_global-1.  The result equals
 * rows [row0, row0+H_band) of gc_filter on the whole image.  Errors as gc_filter, plus
 * GC_ENCCL.  Argument errors are returned before any NCCL call; an error after that
 * (allocation, NCCL) leaves the peers' exchange incomplete: gc_comm_wait detects it.
 */
gc_status gc_bilateral_band(const float* band, int H_band, int W, int H_global, int row0,
                            float sigma_s, float sigma_r, int N, float* out, void* comm,
                            void* stream);

/* gc_filter_band — gc_bilateral_band with the full parameter struct (operator, caller
   coefficients, guard counter, timing events recorded around the two filter passes). */
gc_status gc_filter_band(const float* band, int H_band, int W, int H_global, int row0,
                         const gc_params* p, float* out, void* comm, void* stream);

/*
 * gc_debug_oob_count — bounds-check builds only (libgc_check.so, compiled with
 * -DGC_BOUNDS_CHECK: every global-memory access of the kernels is checked against the call's
 * input segments, plane / scratch buffer, output and taps, since compute-sanitizer is not
 * available on the B200 pool).  Synchronises the device, stores the number of out-of-bounds
 * accesses counted since the last call in *count and resets it.  GC_ERANGE in the product
 * library (no checks compiled in), GC_EINVAL if count is NULL.
 */
gc_status gc_debug_oob_count(unsigned long long* count);

/* gc_debug_oob_selftest — bounds-check builds only: launches a kernel that checks one address
   just past a scratch region and one inside it (no memory access), so that the next
   gc_debug_oob_count reports exactly 1 — the positive control of the checks.  GC_ERANGE in the
   product library. */
gc_status gc_debug_oob_selftest(void);

/*
 * gc_scratch_trim — release reserved stream-ordered scratch of libgc's private memory pool
 * of the current device back to the driver, keeping at most keep_bytes reserved.  libgc
 * never uses the device's default pool; by default its pool keeps freed scratch (the c5
 * plane buffer is 14 GiB) for the next call.  GC_POOL_RELEASE_BYTES (environment, read once
 * per device) bounds what it keeps.  Call after synchronising the streams libgc used.
 */
gc_status gc_scratch_trim(size_t keep_bytes);

/*
 * gc_filter_window — single-GPU building block of the band path (and of the
 * "virtual band" tests): filters output rows [out_row0, out_row0+out_rows) of a global
 * H_global x W image whose input rows are supplied in up to three device segments
 * (top halo, band, bottom halo), seg_row0[k] = global row of seg[k]'s first row,
 * seg_rows[k] its row count (0 = unused).  Every input row the window needs (after
 * symmetric reflection at rows 0 and H_global-1) must lie in a segment (GC_EINVAL
 * otherwise).  out: out_rows*W fp32.
 */
gc_status gc_filter_window(const float* const seg[3], const int seg_row0[3], const int seg_rows[3],
                           int H_global, int W, int out_row0, int out_rows, const gc_params* p,
                           float* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* GC_H_ */
