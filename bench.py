#!/usr/bin/env python
"""Benchmark of the GCF hot path (libgc, sm_100a) — the driver's contract.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2] [--impl ours|reference]

One "step" = one pass of the whole hot path (centre + N+2 auxiliary planes + N+2
spatial Gaussian filterings + recombination and division) over one
batch of the workload's synthetic input.  Default workload: BASELINE.json configs[1]
(c2: one 1024x1024 Voronoi+texture+noise image, sigma_s=5, sigma_r=20, N=8) at its
stated parameters.  The stated (sigma_r, N) are numerically ill-posed for the method
(R1) but the hot-path work depends only on (H, W, N, sigma_s), so the
throughput is that of the parity-gated twin (sigma_r=70) too.

Prints ONE JSON line on rank 0.  Multi-GPU (torchrun, one rank per GPU, NCCL):
c2/c1/c3 run one replica per rank (weak scaling), c4 shards the 256-image batch,
c5 splits the image into row bands with NCCL halo exchange inside libgc.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "megapixels/sec (fp32, degree N, σs) and % of HBM roofline at 1/2/4/8 B200"
FP32_PEAK_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12   # 74.45: SMs x FP32 lanes x 2 x max SM clock


def _hbm_peak():
    """Measured HBM copy bandwidth (GB/s) from the driver-written MEASURED_PEAKS.json, else the
    B200_PROFILING.md fallback."""
    try:
        d = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        for k, v in d.items():
            if "hbm" in k.lower() and isinstance(v, (int, float)) and v > 100:
                return float(v)
    except Exception:
        pass
    return 6550.7


HBM_PEAK_GBPS = _hbm_peak()


def _args():
    a = argparse.ArgumentParser()
    a.add_argument("--gpus", type=int, default=1)
    a.add_argument("--steps", type=int, default=200)
    a.add_argument("--warmup", type=int, default=5)
    a.add_argument("--workload", default="c2", choices=["c1", "c2", "c3", "c4", "c5"])
    a.add_argument("--sigma-s", type=float, default=None, help="c3 sweep value (default: first)")
    a.add_argument("--sigma-r", type=float, default=None, help="override (default: stated)")
    a.add_argument("--impl", default="ours", choices=["ours", "reference"])
    a.add_argument("--no-e2e", action="store_true")
    a.add_argument("--batch", type=int, default=None, help="override the batch size (profiling only)")
    a.add_argument("--no-cpu-baseline", action="store_true")
    a.add_argument("--op", type=int, default=0, choices=[0, 1, 2, 3], help="0 auto, 1 FIR, 2 O(1), 3 Deriche (NOT eq. 7)")
    a.add_argument("--fp64", action="store_true", help="binary64 internal arithmetic (GC_PREC_FP64)")
    return a.parse_args()


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ------------------------------------------------------------------ algorithmic work

O1_FLOP_PER_PLANE = 50   # exact-window recursion per plane-sample and pass:
#                          A, B (2 add) + box (2 add, 1 mul) + 5 resonators x (3 FMA + 1 add + 1 FMA)


DR_FLOP_PER_PLANE = 35  # Deriche mode per plane-sample and pass: 2 sections x 4 FMA per direction
#                         (16 FMA = 32 FLOP) + 3 adds (section sums, causal + anticausal)


def resolve_op(op, R):
    """GC_OP_AUTO -> FIR for W_s <= 24, O(1) above (include/gc.h, gc_api.cpp)."""
    return op if op in (1, 2, 3) else (2 if R >= 25 else 1)


def op_flop_per_plane(op, R):
    """Algorithmic FLOP of the spatial operator per plane-pixel and pass: FIR 2(2R+1); O(1) 50;
    Deriche 35 (lead-in samples excluded)."""
    return {1: 2 * (2 * R + 1), 2: O1_FLOP_PER_PLANE, 3: DR_FLOP_PER_PLANE}[op]


def dr_bytes(N, px):
    """Deriche mode, bytes per launch of its two-pass design (NP plane pairs):
    k_row: f read by both sweeps (8) + causal sums written and re-read (16 NP) + planes written (8 NP);
    k_col: planes read by both sweeps (16 NP) + causal sums written and re-read (16 NP) + f + out (8)."""
    NP = (N + 3) // 2
    return {"k_row": px * (8 + 24 * NP), "k_col": px * (8 + 32 * NP)}


def flops_row(N, R, px, op=1):
    """K_row per input pixel: eq. (7) along rows for N+2 planes + plane generation (N+1 mul,
    once per sample for the FIR, for the entering and leaving samples for O(1)) + centring (6)."""
    gen = (N + 1) + 6
    return px * ((N + 2) * op_flop_per_plane(op, R) + (gen if op == 1 else 2 * gen))


def flops_col(N, R, px, op=1):
    """K_col per output pixel: eq. (7) along columns for N+2 planes + eqs. (8)-(10) 6(N+1) + 8."""
    return px * ((N + 2) * op_flop_per_plane(op, R) + 6 * (N + 1) + 8)


# ------------------------------------------------------------------ clocks during the timed region

class ClockSampler:
    def __init__(self, index=0, period=0.005):
        self.samples, self.reasons, self.max_mhz = [], set(), None
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
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in names.items():
                    if isinstance(bit, int) and bit and (r & bit) == bit and bit not in (0,):
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
        bad = [r for r in self.reasons if r not in ("All", "None", "Unknown")]
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "samples": len(s), "reasons": sorted(bad)}


# ------------------------------------------------------------------ CPU oracle leg

def cpu_oracle_sample(cfg, sigma_s, sigma_r, budget_s=12.0):
    """The oracle as it stands, on a bounded row sample of the workload's first image."""
    import oracle
    from synth import config_image
    img = config_image(cfg, index=0)
    H, W = img.shape
    rows_done, t_used, r0 = 0, 0.0, 0
    block = 32
    while t_used < budget_s and rows_done < H:
        rows = [(r0 + k) % H for k in range(block)]
        t0 = time.perf_counter()
        oracle.gc_filter_rows(img, rows, sigma_s, sigma_r, cfg.N)
        t_used += time.perf_counter() - t0
        rows_done += block
        r0 += H // 7 + 1
    mp = rows_done * W / 1e6
    return {"value": mp / t_used, "unit": "MP/s", "cores": 1, "kind": "oracle",
            "sample": f"{rows_done} output rows x {W} px of {cfg.name} image 0 (oracle.gc_filter_rows, numpy fp64, "
                      f"single-threaded; host nproc={os.cpu_count()}), {t_used:.1f} s"}


def run_reference(args, cfg, sigma_s, sigma_r, ws, rank):
    if rank != 0:
        return
    per_step = max(1.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    vals = []
    for i in range(args.warmup + args.steps):
        r = cpu_oracle_sample(cfg, sigma_s, sigma_r, budget_s=per_step)
        if i >= args.warmup:
            vals.append(r)
    v = float(np.median([r["value"] for r in vals]))
    px_step = cfg.batch * cfg.H * cfg.W       # one step = the whole workload; the oracle timed a row sample
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "MP/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": px_step / (v * 1e6) * 1e3,
            "ms_per_step_note": "extrapolated from the sampled rate", "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": _config(cfg, sigma_s, sigma_r, ws),
            "cpu_baseline": {"value": v, "unit": "MP/s", "cores": 1, "kind": "oracle", "sample": vals[-1]["sample"]},
            "e2e": {"value": v, "unit": "MP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _config(cfg, sigma_s, sigma_r, ws):
    par = {"c4": f"batch-shard{ws}", "c5": f"row-bands{ws}"}.get(cfg.name, f"replicas{ws}")
    return {"workload": f"{cfg.name}: {cfg.batch}x{cfg.H}x{cfg.W} {cfg.kind}", "H": cfg.H, "W": cfg.W,
            "batch": cfg.batch, "sigma_s": sigma_s, "sigma_r": sigma_r, "sigma_r_parity_twin": cfg.sigma_r_twin,
            "N": cfg.N, "planes": cfg.N + 2, "radius": math.ceil(3 * sigma_s), "parallelism": par,
            "l2": "flushed before every timed step (256 MiB write)" if cfg.name in ("c1", "c2", "c3")
            else "inputs larger than L2"}


def _bind_to_gpu_numa_node(index):
    """Run this rank on the CPU cores NVML reports as local to its GPU, so the pinned host
    buffers of the e2e leg sit on the GPU's NUMA node (cross-socket PCIe traffic otherwise
    roughly halves the host<->device copy rate).  No-op when NVML or the affinity call fails."""
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


# ------------------------------------------------------------------ our leg

def main():
    args = _args()
    ws, rank, local = _dist()
    from synth import CONFIGS, config_image
    cfg = CONFIGS[args.workload]
    sigma_s = args.sigma_s if args.sigma_s is not None else cfg.sigma_s[0]
    sigma_r = args.sigma_r if args.sigma_r is not None else cfg.sigma_r
    if args.impl == "reference":
        return run_reference(args, cfg, sigma_s, sigma_r, ws, rank)

    _bind_to_gpu_numa_node(local)                 # before any pinned host allocation (e2e leg)
    import torch
    import torch.distributed as dist
    import paper_1605_02178_b200 as gc
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=dev)
    R = math.ceil(3 * sigma_s)

    # ---- inputs resident in HBM before the timed region
    comm = None
    if args.batch is not None:
        import dataclasses
        cfg = dataclasses.replace(cfg, batch=args.batch)
    if cfg.name == "c4":
        per = cfg.batch // ws
        imgs = np.stack([config_image(cfg, index=rank * per + i) for i in range(per)])
        x = torch.from_numpy(imgs).to(dev)
        H, W, B = cfg.H, cfg.W, per
        px_rank = per * H * W
    elif cfg.name == "c5" and ws > 1:
        full = config_image(cfg)
        rows = [cfg.H // ws] * ws
        pl = gc.band_plan(cfg.H, rank, ws, rows, sigma_s)
        x = torch.from_numpy(np.ascontiguousarray(full[pl["row0"]:pl["row0"] + rows[rank]])).to(dev)
        del full
        H, W, B = rows[rank], cfg.W, 1
        px_rank = H * W
        comm = gc.Comm(rank, ws)
        row0 = pl["row0"]
    else:
        x = torch.from_numpy(config_image(cfg)).to(dev)
        H, W, B = cfg.H, cfg.W, 1
        px_rank = H * W
    out = torch.empty_like(x)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev) if cfg.name in ("c1", "c2", "c3") else None
    stream = torch.cuda.current_stream()

    def step(events=None):
        if comm is not None:
            gc.bilateral_band(x, cfg.H, row0, sigma_s, sigma_r, cfg.N, comm, out=out, op=args.op)
        else:
            gc.filter(x, sigma_s, sigma_r, cfg.N, out=out, events=events, op=args.op, fp64=args.fp64)

    for _ in range(args.warmup):
        if flush is not None:
            flush.zero_()
        step()
    torch.cuda.synchronize()

    K = args.steps
    # timed region: the production call (no events inside it, so the column pass overlaps the
    # row pass's tail through programmatic dependent launch); one event pair per step
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(K)]
    torch.cuda.synchronize()
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
        torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    total_ms = sum(e[0].elapsed_time(e[1]) for e in ev)
    # per-kernel durations (roofline): a second, instrumented pass with events between the
    # kernels (cudaEvent_t handles recorded on the launching stream inside libgc)
    row_ms = col_ms = None
    if comm is None:
        K3 = min(K, 50)
        evk = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(K3)]
        for e in evk:                              # materialise the cudaEvent_t handles
            for q in e:
                q.record()
        torch.cuda.synchronize()
        for k in range(K3):
            if flush is not None:
                flush.zero_()
            step(events=evk[k])
        torch.cuda.synchronize()
        row_ms = sum(e[0].elapsed_time(e[1]) for e in evk) / K3
        col_ms = sum(e[1].elapsed_time(e[2]) for e in evk) / K3
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    px_all = px_rank * ws
    value = px_all * K / (total_ms / 1e3) / 1e6

    # ---- e2e: same metric through gc_filter_host with pinned host buffers
    e2e = None
    if not args.no_e2e and comm is None and not args.fp64:
        hin = torch.from_numpy(x.cpu().numpy()).pin_memory()
        hout = torch.empty_like(hin).pin_memory()
        hin_np, hout_np = hin.numpy(), hout.numpy()
        # DMA to freshly pinned host buffers is slow until the host side has warmed them (per-buffer
        # ramps of hundreds of calls on the B200 VMs, profiles/r01_e2e_host_chunks.txt): warm the
        # e2e leg with 0.5 s of calls on the buffers it times
        t_end = time.perf_counter() + 0.5
        for _ in range(max(3, args.warmup)):
            gc.filter_host(hin_np, sigma_s, sigma_r, cfg.N, out=hout_np, op=args.op)
        while time.perf_counter() < t_end:
            gc.filter_host(hin_np, sigma_s, sigma_r, cfg.N, out=hout_np, op=args.op)
        K2 = min(K, 50)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ms = 0.0
        per = []
        for _ in range(K2):
            if flush is not None:
                flush.zero_()
            e0.record()
            gc.filter_host(hin_np, sigma_s, sigma_r, cfg.N, out=hout_np, op=args.op)
            e1.record()
            e1.synchronize()
            per.append(e0.elapsed_time(e1))
            ms += per[-1]
        if os.environ.get("GC_BENCH_E2E_STEPS"):
            print("e2e steps (ms):", " ".join(f"{v:.3f}" for v in per), file=sys.stderr)
        te = torch.tensor([ms], dtype=torch.float64, device=dev)
        if ws > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        nbytes = int(hin.numel() * 4)
        e2e = {"value": px_all * K2 / (float(te.item()) / 1e3) / 1e6, "unit": "MP/s",
               "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes,
               "api": "gc_filter_host (pinned host buffers; H2D + kernels + D2H + stream sync per step)"}

    if rank != 0:
        if ws > 1:
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel (FP32 ALU bound)
    roof = None
    kernels = None
    if row_ms is not None and not args.fp64:      # (fp64 mode: a correctness instrument, no roofline)
        op = resolve_op(args.op, R)
        fr = flops_row(cfg.N, R, B * H * W, op)   # whole-image row pass (in_rows = H)
        fc = flops_col(cfg.N, R, B * H * W, op)
        kernels = {"k_row": {"ms": row_ms, "tflops": fr / row_ms / 1e9},
                   "k_col": {"ms": col_ms, "tflops": fc / col_ms / 1e9}}
        dom = "k_col" if col_ms >= row_ms else "k_row"
        ach = kernels[dom]["tflops"]
        if op == 3:                                # Deriche mode: HBM bytes of the design, too
            db = dr_bytes(cfg.N, B * H * W)
            for k, ms in (("k_row", row_ms), ("k_col", col_ms)):
                kernels[k]["GBps"] = db[k] / ms / 1e6
        traffic = None
        tp = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tp):
            try:
                key = f"{cfg.name}_s{sigma_s:g}_{ {1: 'fir', 2: 'o1', 3: 'deriche'}[op]}:{dom}"
                traffic = json.load(open(tp)).get(key)
            except Exception:
                traffic = None
        roof = {"bound": "alu", "kernel": dom, "achieved": ach, "peak": FP32_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": ach / FP32_PEAK_TFLOPS, "traffic": traffic,
                "peak_source": "derived: 148 SMs x 128 FP32 lanes x 2 FLOP x 1.965 GHz (B200_PROFILING.md unit "
                               "counts; FFMA measured at 125-128 lanes/clk/SM, profiles/r01_ubench_fp32.txt)"}
        if traffic:
            roof["traffic_bytes_per_px"] = traffic / (B * H * W)     # DRAM bytes per output pixel (ncu)
        if op == 3 and kernels[dom]["GBps"] / HBM_PEAK_GBPS > roof["frac"]:
            roof = {"bound": "hbm", "kernel": dom, "achieved": kernels[dom]["GBps"], "peak": HBM_PEAK_GBPS,
                    "unit": "GB/s", "frac": kernels[dom]["GBps"] / HBM_PEAK_GBPS, "traffic": traffic,
                    "peak_source": "MEASURED_PEAKS.json copy bandwidth (DESIGN.md §5.6 bytes per launch)"}
            if traffic:
                roof["traffic_bytes_per_px"] = traffic / (B * H * W)
    ms_step = total_ms / K
    hbm = {"algorithmic_bytes_per_px": 8, "achieved_GBps": 8 * px_rank / (ms_step / 1e3) / 1e9}
    hbm["frac_of_measured"] = hbm["achieved_GBps"] / HBM_PEAK_GBPS
    line = {"metric": METRIC, "value": value, "unit": "MP/s", "n_gpus": ws, "steps": K, "warmup": args.warmup,
            "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong" if cfg.name in ("c4", "c5") else "weak", "vs_baseline": None, "dtype": "f64" if args.fp64 else "f32",
            "data": "synthetic (seeded, synth/images.py)", "config": _config(cfg, sigma_s, sigma_r, ws),
            "roofline": roof, "kernels": kernels, "hbm": hbm, "e2e": e2e,
            "gpu_launches": 2 * K, "clocks": clk.summary(), "impl": "ours", "lib": gc.version(),
            "host_cores": len(os.sched_getaffinity(0))}
    if ws == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_oracle_sample(cfg, sigma_s, sigma_r)
    print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
