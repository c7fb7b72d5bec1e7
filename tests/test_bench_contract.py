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


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "MP/s" and d["value"] > 0
    assert d["metric"] == bench.METRIC and d["higher_is_better"] is True
    assert d["config"]["workload"].startswith("c2") and d["config"]["N"] == 8
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": "MP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_flop_accounting():
    """FIR: 2(2R+1) FLOP per plane-pixel and pass; O(1): 50; Deriche: 35 (N+2 planes)."""
    N, R, px = 8, 15, 1000
    assert bench.op_flop_per_plane(1, R) == 62
    assert bench.flops_row(N, R, px, 1) == px * (10 * 62 + 15)
    assert bench.flops_col(N, R, px, 1) == px * (10 * 62 + 6 * 9 + 8)
    assert bench.flops_col(N, R, px, 2) == px * (10 * 50 + 6 * 9 + 8)
    assert bench.op_flop_per_plane(3, R) == 35
    assert bench.resolve_op(0, 24) == 1 and bench.resolve_op(0, 25) == 2 and bench.resolve_op(3, 5) == 3


@pytest.mark.parametrize("N,NP", [(5, 4), (8, 5), (12, 7)])
def test_deriche_bytes(N, NP):
    b = bench.dr_bytes(N, 1)
    assert (N + 3) // 2 == NP
    assert b == {"k_row": 8 + 24 * NP, "k_col": 8 + 32 * NP}
