"""CPU tests of bench.py's contract pieces that do not need a GPU: the reference arm's JSON
line (the oracle timed on the host) and the algorithmic work/byte accounting behind the
roofline fields."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_default_workload_is_c5():
    """The driver's default bench line runs the largest single-GPU configuration (c5, row bands at
    N > 1) with K=20 / W=5."""
    a = bench._args([])
    assert a.workload == "c5" and a.gpus == 1 and a.steps >= 1 and a.warmup >= 3 and a.impl == "ours"


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0", "--workload", "c2"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "MP/s" and d["value"] > 0
    assert d["metric"] == bench.METRIC and d["higher_is_better"] is True
    assert d["config"]["workload"].startswith("c2") and d["config"]["N"] == 8
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] == len(os.sched_getaffinity(0)) and cb["value"] == d["value"]
    assert cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": "MP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_json_line_alone_on_stdout():
    """Native code writing to fd 1 (NCCL's version banner under NCCL_DEBUG=VERSION) must not reach
    the driver's stdout: after _quiet_stdout only the JSON line does."""
    code = ("import os, sys; sys.path.insert(0, %r); import bench; bench._quiet_stdout(); "
            "os.write(1, b'NCCL version 0.0.0\\n'); print('python noise'); bench._emit({'metric': 'm', 'value': 1.0})"
            % ROOT)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=120, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    assert r.stdout == '{"metric": "m", "value": 1.0}\n'
    assert "NCCL version" in r.stderr and "python noise" in r.stderr


def test_flop_accounting():
    """FIR: 2(2R+1) FLOP per plane-pixel and pass; O(1): 37; Deriche: 35 (N+2 planes)."""
    N, R, px = 8, 15, 1000
    assert bench.op_flop_per_plane(1, R) == 62
    assert bench.flops_row(N, R, px, 1) == px * (10 * 62 + 15)
    assert bench.flops_col(N, R, px, 1) == px * (10 * 62 + 6 * 9 + 8)
    assert bench.flops_col(N, R, px, 2) == px * (10 * 37 + 6 * 9 + 8)
    assert bench.op_flop_per_plane(3, R) == 35
    assert bench.resolve_op(0, 24) == 1 and bench.resolve_op(0, 25) == 2 and bench.resolve_op(3, 5) == 3


@pytest.mark.parametrize("N,NP", [(5, 4), (8, 5), (12, 7)])
def test_deriche_bytes(N, NP):
    b = bench.dr_bytes(N, 1)
    assert (N + 3) // 2 == NP
    assert b == {"k_row": 8 + 24 * NP, "k_col": 8 + 32 * NP}


def test_algorithmic_instruction_count():
    """2(N+2)17 + 5N + 14 instructions per pixel (c2: 394, c5: 550); the column
    pass's share (N+2)17 + 4(N+1) + 6 (c2: 212)."""
    assert bench.alg_instr(8)["total"] == 394 and bench.alg_instr(12)["total"] == 550
    assert bench.alg_instr(8)["k_col"] == 212
    a = bench.alg_instr(12)
    assert a["k_row"] + a["k_col"] == a["total"]
    assert abs(bench.FP32_PEAK_TINSTR - 37.22) < 0.01


def test_roofline_fields():
    r = bench.roofline(12, 48, 2, 16384 * 16384, row_ms=5.0, col_ms=6.0, step_ms=11.0)
    assert r["kernel"] == "k_col" and r["bound"] == "alu"
    assert abs(r["achieved"] - bench.alg_instr(12)["k_col"] * 16384 ** 2 / 6e-3 / 1e12) < 1e-9
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-12
    assert 0 < r["step_frac"] < r["frac"] * 2 and "derived" in r["peak_source"]


def test_roofline_fused_kernel():
    """The small-image FIR path is one kernel (empty "column" interval): its roofline counts the
    whole step's algorithmic instructions against that kernel's time."""
    px = 1024 * 1024
    r = bench.roofline(8, 15, 1, px, row_ms=0.02, col_ms=0.003, step_ms=0.025, fused=True)
    assert r["kernel"] == "k_fused_fir" and r["alg_instr_per_px"] == bench.alg_instr(8)["total"]
    assert abs(r["achieved"] - bench.alg_instr(8)["total"] * px / 2e-5 / 1e12) < 1e-9


@pytest.mark.parametrize("ws", [1, 2, 8])
def test_check_rows_cover_every_seam(ws):
    """The untimed oracle check includes, for every band seam b, rows b-W, b-1, b and b+W-1."""
    from synth import CONFIGS
    cfg = CONFIGS["c5"]
    rows = [cfg.H // ws] * ws
    chk = bench.check_rows(cfg, 16.0, ws, rows)
    b = 0
    for hb in rows[:-1]:
        b += hb
        assert {b - 48, b - 1, b, b + 47} <= set(chk)
    assert 0 in chk and cfg.H - 1 in chk


def test_oracle_check_crop_is_exact():
    """oracle_check's crops reproduce the whole-image oracle (edge and interior rows)."""
    import numpy as np
    import dataclasses

    import oracle
    import synth
    from synth import CONFIGS, config_image
    cfg = dataclasses.replace(CONFIGS["c2"], H=96, W=80)
    img = config_image("c2", H=96, W=80)
    cfg = dataclasses.replace(cfg, gen=dict(cfg.gen, n_seeds=max(1, round(200 * 96 * 80 / 1024 ** 2))))
    rows = [0, 3, 40, 95]
    ref, _ = oracle.gc_filter_rows(img, rows, 5.0, 70.0, 8)
    real = synth.config_image
    try:
        synth.config_image = lambda c, index=0, rows=None: real("c2", index, H=96, W=80, rows=rows)
        chk = bench.oracle_check(cfg, 5.0, 70.0, rows, ref.astype(np.float32), cols=32)
    finally:
        synth.config_image = real
    assert chk["max_abs"] < 1e-4 and chk["pass"]


def test_traffic_share_of_a_rank():
    """traffic.json holds DRAM bytes per launch of the one-GPU workload: a rank's row band (key
    suffix _g<N>) or batch shard takes its pixel share, so bytes per pixel do not change with N."""
    tr = {"c5_s16_o1:k_col": 1000.0, "_source": "s"}
    full = 100
    t1, _ = bench._traffic(tr, "c5_s16_o1", "k_col", full, full)
    t2, src = bench._traffic(tr, "c5_s16_o1_g4", "k_col", full // 4, full)
    assert t1 == 1000.0 and t2 == 250.0 and "share" in src
    assert bench._traffic(tr, "c5_s16_o1", "k_row", full, full) == (None, None)
