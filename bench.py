#!/usr/bin/env python
"""Benchmark of the GCF hot path (libgc, sm_100a) — the driver's contract.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c5] [--impl ours|reference]

One "step" = one pass of the whole hot path (centre + N+2 auxiliary planes + N+2
spatial Gaussian filterings + recombination and division) over one
batch of the workload's synthetic input.

Default workload: c5 — the single 16384x16384 Voronoi image (sigma_s=16, sigma_r=10,
N=12, O(1) operator via GC_OP_AUTO), BASELINE.json's largest single-GPU configuration.
At --gpus 1 one GPU filters the whole image; at --gpus N > 1 the image is split into N
row bands whose 3 sigma_s-row halos of f are exchanged through NCCL inside libgc
(gc_bilateral_band).  `--gpus N` launches itself under torchrun when
WORLD_SIZE is not set (one rank per GPU, NCCL); the line's n_gpus is the number of ranks
that ran.  c4 shards its 256-image batch over the ranks; c1/c2/c3 run one replica per rank.

The stated (sigma_r, N) are numerically ill-posed for the method (R1) but the
hot-path work depends only on (H, W, N, sigma_s): the timed throughput is that of the
parity-gated twin sigma_r too, and an untimed check of sampled output rows (every band
seam at N > 1) against the CPU oracle at the twin sigma_r is printed in the same line.

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import socket
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "megapixels/sec (fp32, degree N, σs) and % of HBM roofline at 1/2/4/8 B200"
SM_COUNT, FP32_LANES, SM_MAX_GHZ = 148, 128, 1.965
FP32_PEAK_TINSTR = SM_COUNT * FP32_LANES * SM_MAX_GHZ / 1e3   # 37.2 T FP32 lane-instructions/s
FP32_PEAK_TFLOPS = 2 * FP32_PEAK_TINSTR                       # 74.45 TFLOP/s (FMA = 2 FLOP)
PEAK_SOURCE = ("derived: 148 SMs x 128 FP32 lanes x 1.965 GHz max SM clock (B200_PROFILING.md unit counts; "
               "FFMA measured at 125-128 lanes/clk/SM, profiles/r01_ubench_fp32.txt); not driver-measured")
C3_SWEEP = (2.0, 5.0, 10.0, 20.0, 40.0)


def _hbm_peak():
    """Measured HBM copy bandwidth (GB/s) from the driver-written MEASURED_PEAKS.json, else the
    B200_PROFILING.md fallback."""
    try:
        d = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        v = d.get("hbm_gbs")
        if isinstance(v, (int, float)) and v > 100:
            return float(v), "MEASURED_PEAKS.json hbm_gbs (measured copy)"
    except Exception:
        pass
    return 6650.0, "B200_PROFILING.md fallback"


HBM_PEAK_GBPS, HBM_PEAK_SOURCE = _hbm_peak()


def _args(argv=None):
    a = argparse.ArgumentParser()
    a.add_argument("--gpus", type=int, default=1)
    a.add_argument("--steps", type=int, default=20)
    a.add_argument("--warmup", type=int, default=5)
    a.add_argument("--workload", default="c5", choices=["c1", "c2", "c3", "c4", "c5"])
    a.add_argument("--sigma-s", type=float, default=None, help="c3 sweep value (default: first)")
    a.add_argument("--sigma-r", type=float, default=None, help="override (default: stated)")
    a.add_argument("--impl", default="ours", choices=["ours", "reference"])
    a.add_argument("--no-e2e", action="store_true")
    a.add_argument("--no-sweep", action="store_true", help="skip the c3 sigma_s sweep key")
    a.add_argument("--no-check", action="store_true", help="skip the sampled oracle check")
    a.add_argument("--batch", type=int, default=None, help="override the batch size (profiling only)")
    a.add_argument("--no-cpu-baseline", action="store_true")
    a.add_argument("--op", type=int, default=0, choices=[0, 1, 2, 3], help="0 auto, 1 FIR, 2 O(1), 3 Deriche (NOT eq. 7)")
    a.add_argument("--fp64", action="store_true", help="binary64 internal arithmetic (GC_PREC_FP64)")
    a.add_argument("--force-bands", action="store_true",
                   help="c5: run the row-band path (NCCL communicator, gc_bilateral_band) even at one rank "
                        "(exercises the N > 1 code path on one GPU; the band is the whole image)")
    return a.parse_args(argv)


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


_JSON_FD = None


def _quiet_stdout():
    """Keep fd 1 for the one JSON line: anything native code writes to stdout (NCCL prints its
    version banner there when NCCL_DEBUG asks for it) goes to stderr instead."""
    global _JSON_FD
    if _JSON_FD is None:
        sys.stdout.flush()
        _JSON_FD = os.dup(1)
        os.dup2(2, 1)


def _emit(line):
    s = json.dumps(line) + "\n"
    if _JSON_FD is None:
        sys.stdout.write(s)
        sys.stdout.flush()
    else:
        sys.stdout.flush()
        os.write(_JSON_FD, s.encode())


def _self_launch(n):
    """`--gpus N` outside torchrun: re-run this command under torchrun with N ranks."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__), *sys.argv[1:]]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


# ------------------------------------------------------------------ algorithmic work

def alg_instr(N):
    """SURVEY §8(d)'s design-independent count of FP32 lane-instructions per output pixel, with the
    paper's cheapest O(1) Gaussian (Deriche 4th order, 17 instructions per plane and pass; P:50,
    P:112): total 2(N+2)17 + 5N + 14; the column pass's share (N+2)17 + 4(N+1) + 6 (a2 vertical +
    the a3 epilogue, §8(a)); the row pass the rest (a1 + a2 horizontal)."""
    total = 2 * (N + 2) * 17 + 5 * N + 14
    col = (N + 2) * 17 + 4 * (N + 1) + 6
    return {"k_row": total - col, "k_col": col, "total": total}


O1_FLOP_PER_PLANE = 37   # exact-window recursion per plane-sample and pass: A, B (2 add) +
#                          box (1 sub + 1 FMA) + 4 resonators x (3 FMA + 1 add) + output (4 add)
DR_FLOP_PER_PLANE = 35   # Deriche mode per plane-sample and pass: 2 sections x 4 FMA per direction
#                          (16 FMA = 32 FLOP) + 3 adds (section sums, causal + anticausal)


def resolve_op(op, R):
    """GC_OP_AUTO -> FIR for W_s <= 24, O(1) above (include/gc.h, gc_api.cpp)."""
    return op if op in (1, 2, 3) else (2 if R >= 25 else 1)


def op_flop_per_plane(op, R):
    """FLOP of the implemented spatial operator per plane-pixel and pass: FIR 2(2R+1); O(1) 37;
    Deriche 35 (lead-in samples excluded)."""
    return {1: 2 * (2 * R + 1), 2: O1_FLOP_PER_PLANE, 3: DR_FLOP_PER_PLANE}[op]


def dr_bytes(N, px):
    """Deriche mode, bytes per launch of its two-pass design (NP plane pairs):
    k_row: f read by both sweeps (8) + causal sums written and re-read (16 NP) + planes written (8 NP);
    k_col: planes read by both sweeps (16 NP) + causal sums written and re-read (16 NP) + f + out (8)."""
    NP = (N + 3) // 2
    return {"k_row": px * (8 + 24 * NP), "k_col": px * (8 + 32 * NP)}


def flops_row(N, R, px, op=1):
    """The design's work in K_row per input pixel: eq. (7) along rows for N+2 planes + plane
    generation (N+1 mul, once per sample for the FIR, for the entering and leaving samples for
    O(1)) + centring (6)."""
    gen = (N + 1) + 6
    return px * ((N + 2) * op_flop_per_plane(op, R) + (gen if op == 1 else 2 * gen))


def flops_col(N, R, px, op=1):
    """The design's work in K_col per output pixel: eq. (7) along columns for N+2 planes +
    eqs. (8)-(10) 6(N+1) + 8."""
    return px * ((N + 2) * op_flop_per_plane(op, R) + 6 * (N + 1) + 8)


def _traffic(tr, key, kern, px, px_full):
    """DRAM bytes of one launch of `kern` covering px pixels, from profiles/traffic.json (values
    are per launch of the one-GPU workload: a rank's shard or row band takes its share)."""
    base = key.rsplit("_g", 1)[0]
    t = tr.get(f"{base}:{kern}")
    if not t:
        return None, None
    src = tr.get("_source_" + base, tr.get("_source"))
    if px_full and px != px_full:
        t = t * px / px_full
        src = "per pixel of %s, scaled to this rank's share (%s)" % (base, src)
    return t, src


def roofline(N, R, op, px, row_ms, col_ms, step_ms, traffic_key=None, fused=False, px_full=None):
    """Roofline of the dominant kernel: `achieved`/`frac` on SURVEY §8(d)'s
    algorithmic instruction count against the derived FP32 ALU peak; `design` = the same kernel's
    implemented FLOP against 74.45 TFLOP/s; `step_frac` = the whole step on the algorithmic count.
    fused: the call ran as the one small-image FIR kernel (gc_filter_kernels == 1, csrc/gc_fused.cu),
    timed by the first event interval; the second is then empty."""
    alg = alg_instr(N)
    if fused:
        # the small-image FIR path (csrc/gc_fused.cu): one kernel does both passes and eqs. (8)-(10)
        dom, ms, alg = "k_fused_fir", row_ms, dict(alg, k_fused_fir=alg["total"])
        design = (flops_row(N, R, px, op) + flops_col(N, R, px, op)) / (ms / 1e3) / 1e12
    else:
        dom = "k_col" if col_ms >= row_ms else "k_row"
        ms = {"k_row": row_ms, "k_col": col_ms}[dom]
        design = (flops_col if dom == "k_col" else flops_row)(N, R, px, op) / (ms / 1e3) / 1e12
    ach = alg[dom] * px / (ms / 1e3) / 1e12
    out = {"bound": "alu", "kernel": dom, "achieved": ach, "peak": FP32_PEAK_TINSTR,
           "unit": "T FP32 instr/s (SURVEY §8(d) algorithmic count)", "frac": ach / FP32_PEAK_TINSTR,
           "alg_instr_per_px": alg[dom], "units_per_launch": px, "peak_source": PEAK_SOURCE,
           "step_frac": alg["total"] * px / (step_ms / 1e3) / 1e12 / FP32_PEAK_TINSTR,
           "design": {"achieved": design, "peak": FP32_PEAK_TFLOPS, "unit": "TFLOP/s",
                      "frac": design / FP32_PEAK_TFLOPS,
                      "basis": "implemented FLOP: " + {1: "FIR 2(2W+1)", 2: "O(1) 37", 3: "Deriche 35"}[op] +
                               " per plane-pixel and pass + generation / recombination"},
           "traffic": None}
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if traffic_key and os.path.exists(tp):
        try:
            tr = json.load(open(tp))
            t, src = _traffic(tr, traffic_key, dom, px, px_full)
            if t:
                out["traffic"] = t
                out["traffic_bytes_per_px"] = t / px
                out["traffic_source"] = src
        except Exception:
            pass
    return out


# ------------------------------------------------------------------ clocks during the timed region

class ClockSampler:
    def __init__(self, index=0, period=0.005):
        self.samples, self.reasons, self.max_mhz, self.power_w = [], set(), None, []
        self.period, self.index = period, index
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nv = nv
            self.h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        except Exception as e:  # pragma: no cover
            self.err = str(e)
        return self

    def _run(self):
        nv = self.nv
        names = {getattr(nv, k): k for k in dir(nv) if k.startswith("nvmlClocksEventReason") or
                 k.startswith("nvmlClocksThrottleReason")}
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                try:
                    self.power_w.append(nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0)
                except Exception:
                    pass
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in names.items():
                    if isinstance(bit, int) and bit and (r & bit) == bit:
                        self.reasons.add(name.replace("nvmlClocksEventReason", "").replace("nvmlClocksThrottleReason", ""))
            except Exception:
                pass
            time.sleep(self.period)

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        s = sorted(self.samples)
        med = s[len(s) // 2] if s else None
        bad = [r for r in self.reasons if r not in ("All", "None", "Unknown", "GpuIdle")]
        pw = sorted(self.power_w)
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "samples": len(s), "reasons": sorted(bad),
                "power_w_median": pw[len(pw) // 2] if pw else None}


# ------------------------------------------------------------------ CPU oracle (cpu_baseline and --impl reference)

CPU_BLOCK_ROWS, CPU_BLOCK_COLS = 32, 2048


def _cpu_blocks(cfg, n):
    """n deterministic sample blocks (row0, col0) of CPU_BLOCK_ROWS x CPU_BLOCK_COLS output pixels of
    image 0, spread over the image (first block at the top-left corner, which includes the
    symmetric extension)."""
    H, W = cfg.H, cfg.W
    bw = min(CPU_BLOCK_COLS, W)
    br = min(CPU_BLOCK_ROWS, H)
    ncol = max(1, W // bw)
    out = []
    for j in range(n):
        r = (j * 2654435761) % max(1, H - br + 1) if j else 0
        c = ((j * 40503) % ncol) * bw if j else 0
        out.append((int(r) // 8 * 8, int(min(c, W - bw))))
    return out


def _cpu_crop(cfg, blk, sigma_s):
    """The oracle's input for one block: output rows/cols plus the W-sample window on every side
    (or the true image edge, where the oracle applies the symmetric extension itself)."""
    from synth import config_image
    R = math.ceil(3 * sigma_s)
    r0, c0 = blk
    br, bw = min(CPU_BLOCK_ROWS, cfg.H), min(CPU_BLOCK_COLS, cfg.W)
    ya, yb = max(0, r0 - R), min(cfg.H, r0 + br + R)
    xa, xb = max(0, c0 - R), min(cfg.W, c0 + bw + R)
    rows = config_image(cfg, index=0, rows=(ya, yb))
    return np.ascontiguousarray(rows[:, xa:xb]), (r0 - ya, c0 - xa, br, bw, ya == 0 and yb == cfg.H, xa, xb)


def _cpu_worker_warm(_):
    import oracle  # noqa: F401
    return os.getpid()


def _cpu_block_work(args):
    """Worker: oracle.gc_filter_rows on one crop (the oracle as it stands, numpy fp64)."""
    crop, (ry, cx, br, bw, _, _, _), sigma_s, sigma_r, N = args
    import oracle
    t0 = time.perf_counter()
    out, _ = oracle.gc_filter_rows(crop, list(range(ry, ry + br)), sigma_s, sigma_r, N)
    dt = time.perf_counter() - t0
    return dt, out[:, cx:cx + bw]


class CpuOracle:
    """The oracle timed on the host cores: a pool of `cores` single-threaded worker processes,
    each running oracle.gc_filter_rows on its own sample block."""

    def __init__(self, cfg, sigma_s, sigma_r, N, cores=None):
        import multiprocessing as mp
        for v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
            os.environ[v] = "1"
        self.cfg, self.sigma_s, self.sigma_r, self.N = cfg, sigma_s, sigma_r, N
        self.cores = cores or len(os.sched_getaffinity(0))
        self.blocks = _cpu_blocks(cfg, self.cores)
        self.crops = [_cpu_crop(cfg, b, sigma_s) for b in self.blocks]
        # forkserver, not fork: the bench process holds a CUDA context and helper threads (NVML
        # sampler, CUDA runtime) whose locks a forked child could inherit mid-operation
        self.pool = mp.get_context("forkserver").Pool(self.cores) if self.cores > 1 else None
        if self.pool:                              # workers import the oracle before any timing
            self.pool.map(_cpu_worker_warm, range(self.cores), chunksize=1)

    def close(self):
        if self.pool:
            self.pool.close()
            self.pool.join()

    def run(self, cores=None):
        """One round: `cores` blocks in parallel (all cores by default). Returns (MP/s, seconds)."""
        n = cores or self.cores
        work = [(c, m, self.sigma_s, self.sigma_r, self.N) for c, m in self.crops[:n]]
        t0 = time.perf_counter()
        if self.pool is None:
            res = [_cpu_block_work(w) for w in work]
        else:
            res = self.pool.map(_cpu_block_work, work, chunksize=1)
        dt = time.perf_counter() - t0
        px = sum(m[2] * m[3] for _, m in self.crops[:n])
        return px / dt / 1e6, dt

    def describe(self, n, rounds, secs):
        br, bw = min(CPU_BLOCK_ROWS, self.cfg.H), min(CPU_BLOCK_COLS, self.cfg.W)
        return (f"{rounds} round(s) of {n} block(s) of {br} output rows x {bw} px of {self.cfg.name} image 0, "
                f"one block per worker process (oracle.gc_filter_rows on the block's input window, numpy fp64, "
                f"single-threaded workers; host nproc={os.cpu_count()}), {secs:.1f} s")


def cpu_baseline(cfg, sigma_s, sigma_r, N, budget_s=12.0):
    """the oracle on all host cores and on one core, each on a bounded sample."""
    co = CpuOracle(cfg, sigma_s, sigma_r, N)
    try:
        vals, t_all, rounds = [], 0.0, 0
        while t_all < budget_s * 0.6 and rounds < 8:
            v, dt = co.run()
            vals.append(v)
            t_all += dt
            rounds += 1
        v1, t1 = co.run(cores=1)
        return {"value": float(np.median(vals)), "unit": "MP/s", "cores": co.cores, "kind": "oracle",
                "sample": co.describe(co.cores, rounds, t_all),
                "single_core": {"value": v1, "unit": "MP/s", "cores": 1, "sample": co.describe(1, 1, t1)}}
    finally:
        co.close()


def run_reference(args, cfg, sigma_s, sigma_r, ws, rank):
    if rank != 0:
        return
    co = CpuOracle(cfg, sigma_s, sigma_r, cfg.N)
    try:
        vals, t_tot = [], 0.0
        for i in range(args.warmup + args.steps):
            v, dt = co.run()
            if i >= args.warmup:
                vals.append(v)
                t_tot += dt
    finally:
        co.close()
    v = float(np.median(vals))
    px_step = cfg.batch * cfg.H * cfg.W       # one step = the whole workload; the oracle timed a sample of it
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "MP/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": px_step / (v * 1e6) * 1e3,
            "ms_per_step_note": "whole-workload time extrapolated from the sampled rate", "higher_is_better": True,
            "scaling": _scaling(cfg), "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, synth/images.py)",
            "config": _config(cfg, sigma_s, sigma_r, ws),
            "cpu_baseline": {"value": v, "unit": "MP/s", "cores": co.cores, "kind": "oracle",
                             "sample": co.describe(co.cores, args.steps, t_tot) + " per timed step"},
            "e2e": {"value": v, "unit": "MP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    _emit(line)


def band_rows_of(H, ws):
    """Row-band split of c5 over ws ranks (sizes differ by at most one row)."""
    return [H // ws + (1 if k < H % ws else 0) for k in range(ws)]


def shard_of(batch, ws, rank):
    """c4 batch sharding: the image indices rank `rank` filters (contiguous, sizes differ by <= 1)."""
    lo = rank * batch // ws
    return list(range(lo, (rank + 1) * batch // ws))


def _scaling(cfg):
    return "strong" if cfg.name in ("c4", "c5") else "weak"


def _config(cfg, sigma_s, sigma_r, ws):
    par = {"c4": f"batch-shard{ws}", "c5": f"row-bands{ws}"}.get(cfg.name, f"replicas{ws}")
    return {"workload": f"{cfg.name}: {cfg.batch}x{cfg.H}x{cfg.W} {cfg.kind}", "H": cfg.H, "W": cfg.W,
            "batch": cfg.batch, "sigma_s": sigma_s, "sigma_r": sigma_r, "sigma_r_parity_twin": cfg.sigma_r_twin,
            "N": cfg.N, "planes": cfg.N + 2, "radius": math.ceil(3 * sigma_s), "parallelism": par,
            "l2": "flushed before every timed step (256 MiB write)" if cfg.name in ("c1", "c2", "c3")
            else "inputs larger than L2 (no flush)"}


def _bind_to_gpu_numa_node(index):
    """Run this rank on the CPU cores NVML reports as local to its GPU, so the pinned host
    buffers of the e2e leg sit on the GPU's NUMA node.  No-op when NVML or the call fails."""
    try:
        import pynvml as nv
        nv.nvmlInit()
        h = nv.nvmlDeviceGetHandleByIndex(index)
        n = (os.cpu_count() + 63) // 64
        words = nv.nvmlDeviceGetCpuAffinity(h, n)
        cores = {64 * w + b for w, m in enumerate(words) for b in range(64) if (m >> b) & 1}
        cores &= set(range(os.cpu_count()))
        if cores:
            os.sched_setaffinity(0, cores)
    except Exception:
        pass


# ------------------------------------------------------------------ sampled oracle check (untimed)

def check_rows(cfg, sigma_s, ws, band_rows):
    """Global output rows checked against the oracle: every band seam b -> {b-W, b-1, b, b+W-1};
    at one rank a spread of rows incl. both image edges."""
    H = cfg.H
    R = math.ceil(3 * sigma_s)
    rows = {0, min(R, H - 1), H - 1}
    if ws > 1:
        b = 0
        for hb in band_rows[:-1]:
            b += hb
            rows |= {b - R, b - 1, b, b + R - 1}
    else:
        rows |= {H // 2 - 1, H // 2, max(0, H - 1 - R)}
    return sorted(r for r in rows if 0 <= r < H)


def oracle_check(cfg, sigma_s, sigma_r, rows, got, cols=512):
    """Compare GPU output rows `got` [len(rows), W] with the oracle on three column windows (left
    edge, centre, right edge) of each row.  The oracle runs on the crop [r-W, r+W] x [c0-W,
    c0+cols+W] clipped to the image: where the crop is clipped it ends at the true image edge,
    where the oracle's own symmetric extension applies, so the crop determines the row exactly."""
    import oracle
    from synth import config_image
    R = math.ceil(3 * sigma_s)
    H, W = cfg.H, cfg.W
    cw = min(cols, W)
    errs = []
    for i, r in enumerate(rows):
        ya, yb = max(0, r - R), min(H, r + R + 1)
        src = config_image(cfg, index=0, rows=(ya, yb))
        for c0 in sorted({0, (W - cw) // 2, W - cw}):
            xa, xb = max(0, c0 - R), min(W, c0 + cw + R)
            ref, _ = oracle.gc_filter_rows(np.ascontiguousarray(src[:, xa:xb]), [r - ya], sigma_s, sigma_r, cfg.N)
            errs.append(np.abs(got[i, c0:c0 + cw].astype(np.float64) - ref[0, c0 - xa:c0 - xa + cw]))
    e = np.concatenate([x.ravel() for x in errs])
    mx, rm = float(e.max()), float(np.sqrt(np.mean(e ** 2)))
    return {"max_abs": mx, "rms": rm, "rows": len(rows), "px": int(e.size), "sigma_r": sigma_r,
            "tol": {"max_abs": 1e-2, "rms": 1e-3}, "pass": bool(mx <= 1e-2 and rm <= 1e-3),
            "what": "GPU output rows at the parity twin sigma_r (untimed run of the same call) vs "
                    "oracle.gc_filter_rows on each row's input window; left-edge, centre and right-edge columns"}


# ------------------------------------------------------------------ our leg

def _events(n):
    import torch
    return [torch.cuda.Event(enable_timing=True) for _ in range(n)]


def c3_sweep(gc, dev, steps, ops=(0, 2)):
    """BASELINE configs[2]: the 4096^2 image at sigma_r=15, N=10 for sigma_s in {2,5,10,20,40};
    Gpx/s per sigma_s (median of `steps` single-call timings, L2 flushed before each) with
    GC_OP_AUTO and with the O(1) operator forced, plus max/min of each (cost
    independent of sigma_s; the paper's Table II analogue)."""
    import torch
    from synth import CONFIGS, config_image
    cfg = CONFIGS["c3"]
    x = torch.from_numpy(config_image(cfg)).to(dev)
    out = torch.empty_like(x)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    res = {"workload": f"c3: 1x{cfg.H}x{cfg.W} voronoi, sigma_r={cfg.sigma_r}, N={cfg.N}", "unit": "Gpx/s"}
    for op in ops:
        vals = {}
        for s in C3_SWEEP:
            for _ in range(3):
                gc.filter(x, s, cfg.sigma_r, cfg.N, out=out, op=op)
            t = []
            for _ in range(steps):
                flush.zero_()
                e0, e1 = _events(2)
                e0.record()
                gc.filter(x, s, cfg.sigma_r, cfg.N, out=out, op=op)
                e1.record()
                e1.synchronize()
                t.append(e0.elapsed_time(e1))
            vals[f"{s:g}"] = cfg.H * cfg.W / (float(np.median(t)) / 1e3) / 1e9
        v = list(vals.values())
        res["auto" if op == 0 else "o1"] = {"by_sigma_s": vals, "max_over_min": max(v) / min(v)}
    del x, out, flush
    return res


def main():
    args = _args()
    ws, rank, local = _dist()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return _self_launch(args.gpus)
    _quiet_stdout()
    from synth import CONFIGS, config_image
    cfg = CONFIGS[args.workload]
    sigma_s = args.sigma_s if args.sigma_s is not None else cfg.sigma_s[0]
    sigma_r = args.sigma_r if args.sigma_r is not None else cfg.sigma_r
    if args.batch is not None:
        import dataclasses
        cfg = dataclasses.replace(cfg, batch=args.batch)
    if args.impl == "reference":
        return run_reference(args, cfg, sigma_s, sigma_r, ws, rank)

    _bind_to_gpu_numa_node(local)                 # before any pinned host allocation (e2e leg)
    import torch
    import torch.distributed as dist
    import paper_1605_02178_b200 as gc
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1 or args.force_bands:
        if ws == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", str(_free_port()))
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=dev)
    R = math.ceil(3 * sigma_s)
    op = resolve_op(args.op, R) if not args.fp64 else 1
    t_gen0 = time.perf_counter()

    # ---- inputs resident in HBM before the timed region (each rank generates only its part)
    comm, row0, band_rows = None, 0, None
    if cfg.name == "c4":
        mine = shard_of(cfg.batch, ws, rank)
        x = torch.from_numpy(np.stack([config_image(cfg, index=i) for i in mine])).to(dev)
        H, W, B = cfg.H, cfg.W, len(mine)
    elif cfg.name == "c5" and (ws > 1 or args.force_bands):
        band_rows = band_rows_of(cfg.H, ws)
        pl = gc.band_plan(cfg.H, rank, ws, band_rows, sigma_s, op=args.op)
        row0 = pl["row0"]
        x = torch.from_numpy(config_image(cfg, rows=(row0, row0 + band_rows[rank]))).to(dev)
        H, W, B = band_rows[rank], cfg.W, 1
        comm = gc.Comm(rank, ws)
    else:
        x = torch.from_numpy(config_image(cfg)).to(dev)
        H, W, B = cfg.H, cfg.W, 1
    gen_s = time.perf_counter() - t_gen0
    px_rank = B * H * W
    out = torch.empty_like(x)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev) if cfg.name in ("c1", "c2", "c3") else None
    stream = torch.cuda.current_stream()

    # kernels per step as libgc reports them (1 = the fused small-image FIR kernel)
    n_kern = 2 if comm is not None else gc.filter_kernels(B, H, W, sigma_s, sigma_r, cfg.N, op=args.op, fp64=args.fp64)
    fused = n_kern == 1

    def step(events=None, sr=sigma_r, dst=out):
        if comm is not None:
            gc.bilateral_band(x, cfg.H, row0, sigma_s, sr, cfg.N, comm, out=dst, op=args.op, events=events)
        else:
            gc.filter(x, sigma_s, sr, cfg.N, out=dst, events=events, op=args.op, fp64=args.fp64)

    def drain(timeout_ms=300000.0):
        if comm is not None:
            comm.wait(stream, timeout_ms)          # NCCL watchdog (gc_comm_wait)
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        if flush is not None:
            flush.zero_()
        step()
    drain()

    K = args.steps
    # timed region: the production call (no events inside it, so the column pass overlaps the
    # row pass's tail through programmatic dependent launch); one event pair per step
    ev = [_events(2) for _ in range(K)]
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(index=local) as clk:
        for k in range(K):
            if flush is not None:
                flush.zero_()
            ev[k][0].record()
            step()
            ev[k][1].record()
        drain()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    total_ms = sum(e[0].elapsed_time(e[1]) for e in ev)

    # per-kernel durations (roofline): a second, instrumented pass with events between the
    # kernels (cudaEvent_t handles recorded on the launching stream inside libgc)
    row_ms = col_ms = xchg_ms = None
    if not args.fp64:
        K3 = min(K, 20)
        evk = [_events(4) for _ in range(K3)]
        for e in evk:                              # materialise the cudaEvent_t handles
            for q in e:
                q.record()
        torch.cuda.synchronize()
        for k in range(K3):
            if flush is not None:
                flush.zero_()
            evk[k][3].record()
            step(events=evk[k][:3])
        drain()
        row_ms = sum(e[0].elapsed_time(e[1]) for e in evk) / K3
        col_ms = sum(e[1].elapsed_time(e[2]) for e in evk) / K3
        xchg_ms = sum(e[3].elapsed_time(e[0]) for e in evk) / K3

    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    px_all = cfg.batch * cfg.H * cfg.W if cfg.name in ("c4", "c5") else px_rank * ws
    value = px_all * K / (total_ms / 1e3) / 1e6

    # ---- e2e: same metric through the public API with pinned host buffers, copies timed
    e2e = None
    if not args.no_e2e and not args.fp64:
        hin = torch.from_numpy(x.cpu().numpy()).pin_memory()
        hout = torch.empty_like(hin).pin_memory()
        K2 = min(K, 10)
        per = []
        if comm is None:
            # gc_filter_host: H2D + kernels + D2H + stream sync inside one library call
            hin_np, hout_np = hin.numpy(), hout.numpy()
            # DMA to freshly pinned host buffers is slow until warmed (profiles/r01_e2e_host_chunks.txt)
            t_end = time.perf_counter() + 0.5
            for _ in range(max(3, args.warmup)):
                gc.filter_host(hin_np, sigma_s, sigma_r, cfg.N, out=hout_np, op=args.op)
            while time.perf_counter() < t_end:
                gc.filter_host(hin_np, sigma_s, sigma_r, cfg.N, out=hout_np, op=args.op)
            api = "gc_filter_host (pinned host buffers; H2D + kernels + D2H + stream sync per step)"
            for _ in range(K2):
                if flush is not None:
                    flush.zero_()
                e0, e1 = _events(2)
                e0.record()
                gc.filter_host(hin_np, sigma_s, sigma_r, cfg.N, out=hout_np, op=args.op)
                e1.record()
                e1.synchronize()
                per.append(e0.elapsed_time(e1))
        else:
            # per rank: H2D of the band from pinned memory, gc_bilateral_band (exchange + filter),
            # D2H of the band's output, all on the rank's stream
            xb, ob = torch.empty_like(x), torch.empty_like(out)
            api = "per rank: H2D of the band (pinned) + gc_bilateral_band (NCCL halo exchange + filter) + D2H"
            for k in range(args.warmup + K2):
                dist.barrier()
                e0, e1 = _events(2)
                e0.record()
                xb.copy_(hin, non_blocking=True)
                gc.bilateral_band(xb, cfg.H, row0, sigma_s, sigma_r, cfg.N, comm, out=ob, op=args.op)
                hout.copy_(ob, non_blocking=True)
                e1.record()
                comm.wait(stream, 300000.0)
                e1.synchronize()
                if k >= args.warmup:
                    per.append(e0.elapsed_time(e1))
            del xb, ob
        te = torch.tensor([sum(per)], dtype=torch.float64, device=dev)
        if ws > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        nbytes = int(hin.numel() * 4)
        e2e = {"value": px_all * K2 / (float(te.item()) / 1e3) / 1e6, "unit": "MP/s",
               "h2d_bytes_per_step": nbytes * ws, "d2h_bytes_per_step": nbytes * ws,
               "ms_per_step": float(te.item()) / K2, "api": api}
        del hin, hout

    # ---- untimed oracle check of sampled rows at the parity twin sigma_r (all band seams)
    check = None
    rows_chk = None
    if not args.no_check and not args.fp64 and op != 3 and cfg.name in ("c2", "c3", "c5"):
        rows_chk = check_rows(cfg, sigma_s, ws, band_rows or [cfg.H])
        twin = torch.empty_like(out)
        step(sr=cfg.sigma_r_twin, dst=twin)
        drain()
        g = torch.zeros((len(rows_chk), W), dtype=torch.float32, device=dev)
        for i, r in enumerate(rows_chk):
            if row0 <= r < row0 + H:
                g[i] = twin[r - row0] if twin.dim() == 2 else twin[0, r - row0]
        if ws > 1:
            dist.all_reduce(g)                     # each checked row is owned by exactly one rank (x + 0 = x)
        got = g.cpu().numpy()
        del twin

    if rank != 0:
        if comm is not None:
            comm.close()
        if dist.is_initialized():
            dist.destroy_process_group()
        return
    if rows_chk is not None:
        check = oracle_check(cfg, sigma_s, cfg.sigma_r_twin, rows_chk, got)
        if ws > 1:
            check["seams"] = [sum(band_rows[:k + 1]) for k in range(ws - 1)]

    ms_step = total_ms / K
    roof = kernels = None
    if row_ms is not None:
        key = f"{cfg.name}_s{sigma_s:g}_{ {1: 'fir', 2: 'o1', 3: 'deriche'}[op]}" + (f"_g{ws}" if comm else "")
        roof = roofline(cfg.N, R, op, px_rank, row_ms, col_ms, ms_step, traffic_key=key, fused=fused,
                        px_full=cfg.batch * cfg.H * cfg.W)
        fr, fc = flops_row(cfg.N, R, px_rank, op), flops_col(cfg.N, R, px_rank, op)
        if fused:
            kernels = {"k_fused_fir": {"ms": row_ms, "design_tflops": (fr + fc) / row_ms / 1e9}}
        else:
            kernels = {"k_row": {"ms": row_ms, "design_tflops": fr / row_ms / 1e9},
                       "k_col": {"ms": col_ms, "design_tflops": fc / col_ms / 1e9}}
        if comm is not None:
            kernels["halo_exchange"] = {"ms": xchg_ms, "bytes_per_neighbour": R * W * 4}
        if op == 3:                                # Deriche mode: the design's HBM bytes too
            db = dr_bytes(cfg.N, px_rank)
            for k, ms in (("k_row", row_ms), ("k_col", col_ms)):
                kernels[k]["GBps"] = db[k] / ms / 1e6
            d = roof["kernel"]
            if kernels[d]["GBps"] / HBM_PEAK_GBPS > roof["frac"]:
                roof.update({"bound": "hbm", "achieved": kernels[d]["GBps"], "peak": HBM_PEAK_GBPS, "unit": "GB/s",
                             "frac": kernels[d]["GBps"] / HBM_PEAK_GBPS, "peak_source": HBM_PEAK_SOURCE})
    hbm = {"algorithmic_bytes_per_px": 8, "achieved_GBps": 8 * px_rank / (ms_step / 1e3) / 1e9,
           "peak_GBps": HBM_PEAK_GBPS, "peak_source": HBM_PEAK_SOURCE}
    hbm["frac_of_measured"] = hbm["achieved_GBps"] / HBM_PEAK_GBPS
    if row_ms is not None and not fused:
        # the DRAM bytes the kernels actually move (ncu, profiles/traffic.json) over this run's kernel
        # times: how close the implementation runs to the HBM roof, beside the algorithmic 8 B/px
        try:
            tr = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
            px_full = cfg.batch * cfg.H * cfg.W
            tt = {k: _traffic(tr, key, k, px_rank, px_full) for k in ("k_row", "k_col")}
            tb = {k: v[0] for k, v in tt.items()}
            if all(tb.values()):
                dm = {k: {"bytes_per_px": tb[k] / px_rank, "GBps": tb[k] / ms / 1e6,
                          "frac_of_measured": tb[k] / ms / 1e6 / HBM_PEAK_GBPS}
                      for k, ms in (("k_row", row_ms), ("k_col", col_ms))}
                step_gbps = (tb["k_row"] + tb["k_col"]) / ms_step / 1e6
                dm["step"] = {"bytes_per_px": (tb["k_row"] + tb["k_col"]) / px_rank, "GBps": step_gbps,
                              "frac_of_measured": step_gbps / HBM_PEAK_GBPS}
                dm["source"] = ("ncu dram bytes per launch (profiles/traffic.json: %s) / CUDA-event kernel times"
                                % tt["k_col"][1])
                hbm["dram_measured"] = dm
        except Exception:
            pass
    csum = clk.summary()
    energy = None
    if csum.get("power_w_median"):
        # board power during the timed region x step time / pixels of the step (this GPU's share)
        energy = {"J_per_Mpx": csum["power_w_median"] * (ms_step / 1e3) / (px_rank / 1e6),
                  "note": "median NVML board power during the timed region; the step is power-capped when "
                          "clocks.reasons lists SwPowerCap"}
    line = {"metric": METRIC, "value": value, "unit": "MP/s", "n_gpus": ws, "steps": K, "warmup": args.warmup,
            "ms_per_step": ms_step, "higher_is_better": True, "scaling": _scaling(cfg), "vs_baseline": None,
            "dtype": "f64" if args.fp64 else "f32", "data": "synthetic (seeded, synth/images.py)",
            "config": _config(cfg, sigma_s, sigma_r, ws), "roofline": roof, "kernels": kernels, "hbm": hbm,
            "e2e": e2e, "gpu_launches": n_kern * K, "clocks": csum, "energy": energy, "impl": "ours", "lib": gc.version(),
            "host_cores": len(os.sched_getaffinity(0)), "input_generation_s": gen_s}
    if check is not None:
        line["oracle_check"] = check
    if comm is not None:
        comm.close()
    if dist.is_initialized():
        dist.destroy_process_group()
    if not args.no_sweep and cfg.name == "c5":
        line["c3_sweep"] = c3_sweep(gc, dev, 10)
    if ws == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg, sigma_s, sigma_r, cfg.N)
    _emit(line)


if __name__ == "__main__":
    sys.exit(main())
