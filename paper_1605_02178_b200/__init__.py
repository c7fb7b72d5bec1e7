"""paper_1605_02178_b200 — Python binding of libgc (the GCF hot path on B200, sm_100a).

Argument marshalling only: every step of the filter runs in the CUDA kernels behind
the C ABI declared in include/gc.h.  PyTorch is used for device memory and streams.
There is no CPU fallback: if libgc.so is missing or cannot be loaded, importing the
compute entry points raises.

Names follow include/gc.h and the paper's notation (sigma_s, sigma_r, N, c_n, mu).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

__all__ = [
    "GCError", "lib", "coeffs", "bilateral", "bilateral_batch", "bilateral_c", "filter",
    "filter_host", "filter_window", "band_plan", "Comm", "bilateral_band", "version",
    "OP_AUTO", "OP_FIR", "OP_O1", "OP_DERICHE", "gaussian", "operator_taps", "bilateral_direct",
    "band_exchange_plan", "filter_band", "scratch_trim", "debug_oob_count", "debug_oob_selftest",
    "filter_kernels",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GC_LIB_PATH") or os.path.join(_HERE, "libgc.so")   # override: A/B timing of builds

OP_AUTO, OP_FIR, OP_O1, OP_DERICHE = 0, 1, 2, 3   # gc_operator (include/gc.h)
PREC_FP32, PREC_FP64 = 0, 1
_STATUS = {0: "GC_OK", 1: "GC_EINVAL", 2: "GC_ERANGE", 3: "GC_ECUDA", 4: "GC_ENOMEM", 5: "GC_ENCCL",
           6: "GC_ETIMEOUT"}


class GCError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        super().__init__(f"{where}: {_STATUS.get(status, status)} ({_lib().gc_status_string(status).decode()})")


class _Params(ctypes.Structure):
    _fields_ = [
        ("N", ctypes.c_int),
        ("sigma_s", ctypes.c_float),
        ("sigma_r", ctypes.c_float),
        ("L", ctypes.c_float),
        ("U", ctypes.c_float),
        ("c", ctypes.POINTER(ctypes.c_double)),
        ("op", ctypes.c_int),
        ("fallback_count", ctypes.c_void_p),
        ("events", ctypes.c_void_p * 3),
        ("precision", ctypes.c_int),
    ]


class _Xfer(ctypes.Structure):
    _fields_ = [("peer", ctypes.c_int), ("send_offset", ctypes.c_size_t), ("count", ctypes.c_size_t),
                ("recv_row0", ctypes.c_int)]


_LIB = None


def _lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libgc.so not built ({LIB_PATH}); run `python -m paper_1605_02178_b200.build`")
        L = ctypes.CDLL(LIB_PATH)
        vp, i, f, d = ctypes.c_void_p, ctypes.c_int, ctypes.c_float, ctypes.c_double
        ip = ctypes.POINTER(ctypes.c_int)
        L.gc_status_string.restype = ctypes.c_char_p
        L.gc_status_string.argtypes = [i]
        L.gc_version.restype = ctypes.c_char_p
        L.gc_coeffs.argtypes = [i, d, d, d, ctypes.POINTER(d), ctypes.POINTER(d)]
        L.gc_bilateral.argtypes = [vp, i, i, f, f, i, vp, vp]
        L.gc_bilateral_batch.argtypes = [vp, i, i, i, f, f, i, vp, vp]
        L.gc_bilateral_c.argtypes = [vp, i, i, f, f, i, ctypes.POINTER(d), vp, vp]
        L.gc_params_init.argtypes = [ctypes.POINTER(_Params), i, f, f]
        L.gc_params_init.restype = None
        L.gc_filter.argtypes = [vp, i, i, i, ctypes.POINTER(_Params), vp, vp]
        L.gc_filter_host.argtypes = [vp, i, i, i, ctypes.POINTER(_Params), vp, vp]
        L.gc_filter_kernels.argtypes = [i, i, i, ctypes.POINTER(_Params), ip]
        L.gc_filter_window.argtypes = [ctypes.POINTER(vp), ip, ip, i, i, i, i, ctypes.POINTER(_Params), vp, vp]
        L.gc_gaussian.argtypes = [vp, i, i, i, f, i, vp, vp]
        L.gc_bilateral_direct.argtypes = [vp, i, i, i, f, f, vp, vp]
        L.gc_operator_taps.argtypes = [f, i, ctypes.POINTER(d), ip]
        L.gc_band_plan.argtypes = [i, i, i, ip, f, i, ip, ip, ip, ip, ip]
        L.gc_band_exchange_plan.argtypes = [i, i, i, i, i, i, f, i, ctypes.POINTER(_Xfer), ip, ip]
        L.gc_comm_wait.argtypes = [vp, vp, d]
        L.gc_filter_band.argtypes = [vp, i, i, i, i, ctypes.POINTER(_Params), vp, vp, vp]
        L.gc_scratch_trim.argtypes = [ctypes.c_size_t]
        L.gc_debug_oob_count.argtypes = [ctypes.POINTER(ctypes.c_ulonglong)]
        L.gc_debug_oob_selftest.argtypes = []
        L.gc_comm_unique_id.argtypes = [ctypes.c_char_p]
        L.gc_comm_init.argtypes = [i, i, ctypes.c_char_p, ctypes.POINTER(vp)]
        L.gc_comm_destroy.argtypes = [vp]
        L.gc_bilateral_band.argtypes = [vp, i, i, i, i, f, f, i, vp, vp, vp]
        for name in ["gc_coeffs", "gc_bilateral", "gc_bilateral_batch", "gc_bilateral_c", "gc_filter",
                     "gc_filter_host", "gc_filter_window", "gc_band_plan", "gc_comm_unique_id",
                     "gc_comm_init", "gc_comm_destroy", "gc_bilateral_band", "gc_gaussian", "gc_operator_taps",
                     "gc_bilateral_direct", "gc_band_exchange_plan", "gc_comm_wait", "gc_filter_band",
                     "gc_scratch_trim", "gc_debug_oob_count", "gc_debug_oob_selftest", "gc_filter_kernels"]:
            getattr(L, name).restype = ctypes.c_int
        _LIB = L
    return _LIB


lib = _lib


def _check(st, where):
    if st != 0:
        raise GCError(st, where)


def version() -> str:
    return _lib().gc_version().decode()


def coeffs(N: int, sigma_r: float, L: float = 0.0, U: float = 255.0):
    """c_0..c_N of eq. (19) (binary64, computed in libgc's multiprecision) and mu."""
    c = (ctypes.c_double * (N + 1))()
    mu = ctypes.c_double()
    _check(_lib().gc_coeffs(int(N), float(sigma_r), float(L), float(U), c, ctypes.byref(mu)), "gc_coeffs")
    return np.array(c[:], dtype=np.float64), mu.value


def _params(N, sigma_s, sigma_r, L=0.0, U=255.0, c=None, op=OP_AUTO, fallback=None, events=None, fp64=False):
    p = _Params()
    _lib().gc_params_init(ctypes.byref(p), int(N), float(sigma_s), float(sigma_r))
    p.L, p.U, p.op = float(L), float(U), int(op)
    p.precision = PREC_FP64 if fp64 else PREC_FP32
    keep = None
    if c is not None:
        keep = (ctypes.c_double * (N + 1))(*[float(v) for v in c])
        p.c = ctypes.cast(keep, ctypes.POINTER(ctypes.c_double))
    if fallback is not None:
        p.fallback_count = fallback.data_ptr()
    if events is not None:                    # three torch.cuda.Event (recorded once already)
        for i, ev in enumerate(events):
            p.events[i] = ev.cuda_event
    return p, keep


def _stream(stream, device=None):
    """The cudaStream_t to enqueue on: `stream`, else the current stream of `device` (the
    input tensor's device, on which libgc allocates and launches)."""
    import torch
    if stream is not None:
        if device is not None and stream.device != device:
            raise ValueError(f"stream is on {stream.device}, the tensors on {device}")
        return ctypes.c_void_p(stream.cuda_stream)
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _dev_f32(t, name):
    import torch
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()):
        raise TypeError(f"{name} must be a contiguous float32 CUDA tensor")
    return ctypes.c_void_p(t.data_ptr())


def _out_like(out, shape, device, name="out"):
    """Allocate `out`, or check a caller-supplied one: contiguous float32 CUDA tensor of
    exactly `shape` on `device` (libgc writes prod(shape) floats through the pointer)."""
    import torch
    if out is None:
        return torch.empty(tuple(shape), dtype=torch.float32, device=device)
    _dev_f32(out, name)
    if tuple(out.shape) != tuple(shape):
        raise ValueError(f"{name} has shape {tuple(out.shape)}, expected {tuple(shape)}")
    if out.device != device:
        raise ValueError(f"{name} is on {out.device}, the input on {device}")
    return out


class _on_device:
    """Run a libgc call with `device` current (libgc allocates scratch and launches on the
    current device)."""

    def __init__(self, device):
        import torch
        self.ctx = torch.cuda.device(device)

    def __enter__(self):
        self.ctx.__enter__()

    def __exit__(self, *a):
        self.ctx.__exit__(*a)


def _bhw(img):
    if img.dim() == 2:
        return 1, img.shape[0], img.shape[1]
    if img.dim() == 3:
        return tuple(img.shape)
    raise ValueError("img must be [H, W] or [B, H, W]")


def filter(img, sigma_s, sigma_r, N, c=None, L=0.0, U=255.0, out=None, op=OP_AUTO, fallback=None, stream=None,
           events=None, fp64=False):
    """GCF of a [H, W] or [B, H, W] float32 CUDA tensor (gc_filter).  Asynchronous on `stream`.

    c: optional caller coefficients c_0..c_N (e.g. 1/n! = GPF); fallback: optional int64
    CUDA tensor of one element that receives the number of guarded pixels (R8); fp64: binary64
    internal arithmetic (GC_PREC_FP64)."""
    B, H, W = _bhw(img)
    iv = _dev_f32(img, "img")
    out = _out_like(out, img.shape, img.device)
    if fallback is not None and not (fallback.is_cuda and fallback.device == img.device and fallback.numel() >= 1
                                     and fallback.element_size() == 8):
        raise TypeError("fallback must be a 64-bit CUDA tensor on the input's device")
    p, keep = _params(N, sigma_s, sigma_r, L, U, c, op, fallback, events, fp64)
    with _on_device(img.device):
        _check(_lib().gc_filter(iv, B, H, W, ctypes.byref(p), _dev_f32(out, "out"), _stream(stream, img.device)),
               "gc_filter")
    del keep
    return out


def filter_kernels(B, H, W, sigma_s, sigma_r, N, c=None, L=0.0, U=255.0, op=OP_AUTO, fp64=False):
    """gc_filter_kernels: kernels gc_filter launches for this shape and these parameters (1 = the
    fused small-image FIR kernel, 2 = the two passes).  Host only."""
    p, keep = _params(N, sigma_s, sigma_r, L, U, c, op, None, None, fp64)
    n = ctypes.c_int(0)
    _check(_lib().gc_filter_kernels(int(B), int(H), int(W), ctypes.byref(p), ctypes.byref(n)), "gc_filter_kernels")
    del keep
    return int(n.value)


def gaussian(img, sigma_s, op=OP_AUTO, out=None, stream=None):
    """gc_gaussian: eq. (7) alone on a [H, W] or [B, H, W] float32 CUDA tensor (operator `op`)."""
    B, H, W = _bhw(img)
    iv = _dev_f32(img, "img")
    out = _out_like(out, img.shape, img.device)
    with _on_device(img.device):
        _check(_lib().gc_gaussian(iv, B, H, W, float(sigma_s), int(op), _dev_f32(out, "out"),
                                  _stream(stream, img.device)), "gc_gaussian")
    return out


def bilateral_direct(img, sigma_s, sigma_r, out=None, stream=None):
    """gc_bilateral_direct: eq. (1) itself on a [H, W] or [B, H, W] float32 CUDA tensor (reference)."""
    B, H, W = _bhw(img)
    iv = _dev_f32(img, "img")
    out = _out_like(out, img.shape, img.device)
    with _on_device(img.device):
        _check(_lib().gc_bilateral_direct(iv, B, H, W, float(sigma_s), float(sigma_r), _dev_f32(out, "out"),
                                          _stream(stream, img.device)), "gc_bilateral_direct")
    return out


def operator_taps(sigma_s, op=OP_AUTO):
    """gc_operator_taps (host only): the 1-D impulse response k[-W..W] operator `op` applies."""
    Wr = ctypes.c_int()
    _check(_lib().gc_operator_taps(float(sigma_s), int(op), None, ctypes.byref(Wr)), "gc_operator_taps")
    t = (ctypes.c_double * (2 * Wr.value + 1))()
    _check(_lib().gc_operator_taps(float(sigma_s), int(op), t, ctypes.byref(Wr)), "gc_operator_taps")
    return np.array(t[:], dtype=np.float64)


def bilateral(img, sigma_s, sigma_r, N, out=None, stream=None):
    """gc_bilateral: one [H, W] image, Chebyshev coefficients, [L, U] = [0, 255]."""
    H, W = img.shape
    iv = _dev_f32(img, "img")
    out = _out_like(out, img.shape, img.device)
    with _on_device(img.device):
        _check(_lib().gc_bilateral(iv, H, W, float(sigma_s), float(sigma_r), int(N), _dev_f32(out, "out"),
                                   _stream(stream, img.device)), "gc_bilateral")
    return out


def bilateral_batch(imgs, sigma_s, sigma_r, N, out=None, stream=None):
    """gc_bilateral_batch: [B, H, W] images with one parameter set."""
    B, H, W = imgs.shape
    iv = _dev_f32(imgs, "imgs")
    out = _out_like(out, imgs.shape, imgs.device)
    with _on_device(imgs.device):
        _check(_lib().gc_bilateral_batch(iv, B, H, W, float(sigma_s), float(sigma_r), int(N), _dev_f32(out, "out"),
                                         _stream(stream, imgs.device)), "gc_bilateral_batch")
    return out


def bilateral_c(img, sigma_s, sigma_r, N, c, out=None, stream=None):
    """gc_bilateral_c: caller coefficients c_0..c_N (e.g. Taylor 1/n! -> GPF)."""
    H, W = img.shape
    iv = _dev_f32(img, "img")
    out = _out_like(out, img.shape, img.device)
    if len(c) != N + 1:
        raise ValueError("need N+1 coefficients")
    cc = (ctypes.c_double * (N + 1))(*[float(v) for v in c])
    with _on_device(img.device):
        _check(_lib().gc_bilateral_c(iv, H, W, float(sigma_s), float(sigma_r), int(N), cc, _dev_f32(out, "out"),
                                     _stream(stream, img.device)), "gc_bilateral_c")
    return out


def filter_host(img: np.ndarray, sigma_s, sigma_r, N, c=None, L=0.0, U=255.0, out: np.ndarray | None = None,
                stream=None, op=OP_AUTO, device=None):
    """gc_filter_host: host float32 arrays in and out (pinned recommended); synchronous.
    Runs on `device` (default: the current CUDA device)."""
    import torch
    if not (isinstance(img, np.ndarray) and img.dtype == np.float32 and img.flags.c_contiguous):
        raise TypeError("img must be a C-contiguous float32 array")
    if img.ndim not in (2, 3):
        raise ValueError("img must be [H, W] or [B, H, W]")
    B, H, W = (1, *img.shape) if img.ndim == 2 else img.shape
    if out is None:
        out = np.empty_like(img)
    elif not (isinstance(out, np.ndarray) and out.dtype == np.float32 and out.flags.c_contiguous
              and out.flags.writeable and out.shape == img.shape):
        raise TypeError(f"out must be a writeable C-contiguous float32 array of shape {img.shape}")
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    p, keep = _params(N, sigma_s, sigma_r, L, U, c, op)
    with _on_device(dev):
        _check(_lib().gc_filter_host(ctypes.c_void_p(img.ctypes.data), B, H, W, ctypes.byref(p),
                                     ctypes.c_void_p(out.ctypes.data), _stream(stream, dev)), "gc_filter_host")
    del keep
    return out


def filter_window(segs, H_global, out_row0, out_rows, sigma_s, sigma_r, N, c=None, out=None, stream=None,
                  op=OP_AUTO):
    """gc_filter_window: segs = list of up to 3 (tensor [rows, W], global_row0)."""
    if not 1 <= len(segs) <= 3:
        raise ValueError("1..3 segments")
    W = segs[0][0].shape[1]
    dev = segs[0][0].device
    ptrs = (ctypes.c_void_p * 3)()
    r0 = (ctypes.c_int * 3)()
    nr = (ctypes.c_int * 3)()
    for k, (t, g0) in enumerate(segs):
        if t.dim() != 2 or t.shape[1] != W or t.device != dev:
            raise ValueError("segments must be [rows, W] tensors on one device")
        ptrs[k] = _dev_f32(t, "seg").value
        r0[k], nr[k] = int(g0), int(t.shape[0])
    out = _out_like(out, (out_rows, W), dev)
    p, keep = _params(N, sigma_s, sigma_r, c=c, op=op)
    with _on_device(dev):
        _check(_lib().gc_filter_window(ptrs, r0, nr, int(H_global), int(W), int(out_row0), int(out_rows),
                                       ctypes.byref(p), _dev_f32(out, "out"), _stream(stream, dev)),
               "gc_filter_window")
    del keep
    return out


def band_plan(H_global, rank, world, band_rows, sigma_s, op=OP_AUTO):
    """gc_band_plan (host only): dict(row0, top0, top_rows, bot0, bot_rows) for `rank`."""
    if len(band_rows) != world:
        raise ValueError("band_rows must have `world` entries")
    br = (ctypes.c_int * world)(*[int(v) for v in band_rows])
    o = [ctypes.c_int() for _ in range(5)]
    _check(_lib().gc_band_plan(int(H_global), int(rank), int(world), br, float(sigma_s), int(op),
                               *[ctypes.byref(v) for v in o]), "gc_band_plan")
    return dict(zip(["row0", "top0", "top_rows", "bot0", "bot_rows"], [v.value for v in o]))


def band_exchange_plan(H_band, W, H_global, row0, rank, world, sigma_s, op=OP_AUTO):
    """gc_band_exchange_plan (host only): what gc_filter_band sends/receives and filters.

    Returns (xfers, segs): xfers = [dict(peer, send_offset, count, recv_row0)] for rank-1 and
    rank+1 (peer -1: none), segs = [(seg_row0, seg_rows)] x 3 (top halo, band, bottom halo)."""
    x = (_Xfer * 2)()
    sr0 = (ctypes.c_int * 3)()
    srn = (ctypes.c_int * 3)()
    _check(_lib().gc_band_exchange_plan(int(H_band), int(W), int(H_global), int(row0), int(rank), int(world),
                                        float(sigma_s), int(op), x, sr0, srn), "gc_band_exchange_plan")
    xf = [dict(peer=v.peer, send_offset=v.send_offset, count=v.count, recv_row0=v.recv_row0) for v in x]
    return xf, [(sr0[k], srn[k]) for k in range(3)]


class Comm:
    """libgc-owned NCCL communicator; the 128-byte unique id is broadcast with torch.distributed."""

    def __init__(self, rank: int, world: int, group=None):
        import torch
        import torch.distributed as dist
        buf = torch.zeros(128, dtype=torch.uint8)
        if rank == 0:
            raw = ctypes.create_string_buffer(128)
            _check(_lib().gc_comm_unique_id(raw), "gc_comm_unique_id")
            buf = torch.frombuffer(bytearray(raw.raw), dtype=torch.uint8).clone()
        if dist.get_backend(group) == "nccl":
            buf = buf.cuda()
        dist.broadcast(buf, src=0, group=group)
        ident = bytes(buf.cpu().numpy().tobytes())
        self.rank, self.world = rank, world
        self.handle = ctypes.c_void_p()
        _check(_lib().gc_comm_init(int(rank), int(world), ident, ctypes.byref(self.handle)), "gc_comm_init")

    def wait(self, stream=None, timeout_ms=60000.0):
        """gc_comm_wait: block until `stream` is idle, polling NCCL asynchronous errors; aborts
        the communicator and raises GCError (GC_ENCCL / GC_ETIMEOUT) on failure or timeout."""
        _check(_lib().gc_comm_wait(self.handle, _stream(stream), float(timeout_ms)), "gc_comm_wait")

    def close(self):
        if self.handle:
            _check(_lib().gc_comm_destroy(self.handle), "gc_comm_destroy")
            self.handle = ctypes.c_void_p()


def bilateral_band(band, H_global, row0, sigma_s, sigma_r, N, comm: Comm, c=None, out=None, stream=None,
                   op=OP_AUTO, events=None):
    """This rank's rows [row0, row0+H_band) of the GCF of a row-sharded image.

    With the defaults (no c, op AUTO, no events) this is SURVEY §8(b)'s gc_bilateral_band;
    otherwise gc_filter_band with the full parameter struct."""
    H_band, W = band.shape
    bv = _dev_f32(band, "band")
    out = _out_like(out, band.shape, band.device)
    with _on_device(band.device):
        st = _stream(stream, band.device)
        if c is None and op == OP_AUTO and events is None:
            _check(_lib().gc_bilateral_band(bv, H_band, W, int(H_global), int(row0), float(sigma_s), float(sigma_r),
                                            int(N), _dev_f32(out, "out"), comm.handle, st), "gc_bilateral_band")
        else:
            p, keep = _params(N, sigma_s, sigma_r, c=c, op=op, events=events)
            _check(_lib().gc_filter_band(bv, H_band, W, int(H_global), int(row0), ctypes.byref(p),
                                         _dev_f32(out, "out"), comm.handle, st), "gc_filter_band")
            del keep
    return out


filter_band = bilateral_band


def scratch_trim(keep_bytes: int = 0, device=None):
    """gc_scratch_trim: release libgc's reserved stream-ordered scratch on `device`."""
    import torch
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    with _on_device(dev):
        _check(_lib().gc_scratch_trim(int(keep_bytes)), "gc_scratch_trim")


def debug_oob_count():
    """gc_debug_oob_count: out-of-bounds device accesses counted since the last call (bounds-check
    build libgc_check.so only; raises GCError(GC_ERANGE) on the product library)."""
    c = ctypes.c_ulonglong()
    _check(_lib().gc_debug_oob_count(ctypes.byref(c)), "gc_debug_oob_count")
    return int(c.value)


def debug_oob_selftest():
    """gc_debug_oob_selftest: positive control — the next debug_oob_count() returns exactly 1."""
    _check(_lib().gc_debug_oob_selftest(), "gc_debug_oob_selftest")
