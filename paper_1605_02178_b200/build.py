"""In-tree build of libgc.so (sm_100a) with nvcc.

    python -m paper_1605_02178_b200.build          # incremental
    python -m paper_1605_02178_b200.build --clean  # rebuild everything

Objects go to build/ at the repo root; the shared library is written next to this
file (paper_1605_02178_b200/libgc.so) so it travels with `gpurun` snapshots.  A second
library, libgc_check.so (objects in build_check/), is the same code compiled with
-DGC_BOUNDS_CHECK: every global-memory access of the kernels is range-checked and violations
are counted (gc_debug_oob_count) — the test suite's substitute for compute-sanitizer, which
the B200 pool does not offer.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "libgc.so")
VARIANTS = {  # library -> (object directory, extra flags)
    LIB: (BUILD, []),
    os.path.join(PKG, "libgc_check.so"): (os.path.join(ROOT, "build_check"), ["-DGC_BOUNDS_CHECK"]),
}

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", f"-I{INCLUDE}"]


def _nccl_dirs():
    try:
        import nvidia.nccl as n  # torch's NCCL 2.28 wheel
        base = os.path.dirname(n.__file__) if getattr(n, "__file__", None) else list(n.__path__)[0]
        inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    except Exception:
        pass
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def _sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cpp")))


def _headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    return hs + [os.path.join(INCLUDE, "gc.h")]


def _obj(src, bdir):
    return os.path.join(bdir, os.path.basename(src) + ".o")


def _compile(src, nccl_inc, verbose, bdir, extra):
    obj = _obj(src, bdir)
    cmd = [NVCC, *ARCH, *COMMON, *extra, f"-I{nccl_inc}", "-c", src, "-o", obj]
    if src.endswith(".cu") and verbose:
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj, r.stderr


def _build_one(lib, bdir, extra, clean, verbose, nccl_inc, nccl_lib):
    if clean and os.path.isdir(bdir):
        shutil.rmtree(bdir)
    os.makedirs(bdir, exist_ok=True)
    srcs = _sources()
    newest_hdr = max(os.path.getmtime(h) for h in _headers())
    todo = [s for s in srcs if not os.path.exists(_obj(s, bdir))
            or os.path.getmtime(_obj(s, bdir)) < max(os.path.getmtime(s), newest_hdr)]
    with cf.ThreadPoolExecutor(max_workers=max(1, min(len(todo), os.cpu_count() or 1))) as ex:
        for obj, log in ex.map(lambda s: _compile(s, nccl_inc, verbose, bdir, extra), todo):
            if verbose and log:
                print(log, file=sys.stderr)
    objs = [_obj(s, bdir) for s in srcs]
    if todo or not os.path.exists(lib) or os.path.getmtime(lib) < max(os.path.getmtime(o) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", lib, *objs, f"-L{nccl_lib}", "-l:libnccl.so.2",
               "-Xlinker", f"-rpath,{nccl_lib}", "-lcudart_static", "-lrt", "-ldl", "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return lib


def build(clean: bool = False, verbose: bool = False, check: bool = True) -> str:
    """Build libgc.so (and, unless check=False, the bounds-checked libgc_check.so)."""
    nccl_inc, nccl_lib = _nccl_dirs()
    for lib, (bdir, extra) in VARIANTS.items():
        if lib != LIB and not check:
            continue
        _build_one(lib, bdir, extra, clean, verbose, nccl_inc, nccl_lib)
    return LIB


if __name__ == "__main__":
    print(build(clean="--clean" in sys.argv, verbose="-v" in sys.argv, check="--no-check" not in sys.argv))
