"""In-tree build of libgc.so (sm_100a) with nvcc.

    python -m paper_1605_02178_b200.build          # incremental
    python -m paper_1605_02178_b200.build --clean  # rebuild everything

Objects go to build/ at the repo root; the shared library is written next to this
file (paper_1605_02178_b200/libgc.so) so it travels with `gpurun` snapshots.
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


def _obj(src):
    return os.path.join(BUILD, os.path.basename(src) + ".o")


def _compile(src, nccl_inc, verbose):
    obj = _obj(src)
    cmd = [NVCC, *ARCH, *COMMON, f"-I{nccl_inc}", "-c", src, "-o", obj]
    if src.endswith(".cu"):
        cmd.insert(1, "-Xptxas=-v") if verbose else None
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj, r.stderr


def build(clean: bool = False, verbose: bool = False) -> str:
    if clean and os.path.isdir(BUILD):
        shutil.rmtree(BUILD)
    os.makedirs(BUILD, exist_ok=True)
    nccl_inc, nccl_lib = _nccl_dirs()
    srcs = _sources()
    newest_hdr = max(os.path.getmtime(h) for h in _headers())
    todo = [s for s in srcs if not os.path.exists(_obj(s))
            or os.path.getmtime(_obj(s)) < max(os.path.getmtime(s), newest_hdr)]
    with cf.ThreadPoolExecutor(max_workers=max(1, min(len(todo), os.cpu_count() or 1))) as ex:
        for obj, log in ex.map(lambda s: _compile(s, nccl_inc, verbose), todo):
            if verbose and log:
                print(log, file=sys.stderr)
    objs = [_obj(s) for s in srcs]
    if todo or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, f"-L{nccl_lib}", "-l:libnccl.so.2",
               "-Xlinker", f"-rpath,{nccl_lib}", "-lcudart_static", "-lrt", "-ldl", "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(clean="--clean" in sys.argv, verbose="-v" in sys.argv))
