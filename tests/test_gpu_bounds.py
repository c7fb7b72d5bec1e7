"""Memory-safety checks of every device path (the substitute for compute-sanitizer, which the
B200 pool does not offer).  libgc_check.so is libgc compiled with
-DGC_BOUNDS_CHECK: every global-memory access of the FIR, O(1), Deriche and binary64 kernels is
range-checked against the call's input segments, plane / scratch buffer, output and taps, and
violations are counted.  tools/sanitize_cases.py drives small cases of every path through it
(odd / even / 1-pixel widths, batches, interior row windows of the band path, the e2e host
pipeline, large N) and checks NaN guard margins around outputs."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECK_LIB = os.path.join(ROOT, "paper_1605_02178_b200", "libgc_check.so")

pytestmark = pytest.mark.gpu


def _run(code):
    env = dict(os.environ, GC_LIB_PATH=CHECK_LIB)
    return subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600, cwd=ROOT,
                          env=env)


def test_bounds_checks_catch_a_violation(cuda_device):
    """Positive control: the self-test kernel makes exactly one out-of-bounds check fail."""
    assert os.path.exists(CHECK_LIB), "build libgc_check.so (python -m paper_1605_02178_b200.build)"
    r = _run("import paper_1605_02178_b200 as gc; gc.debug_oob_count(); gc.debug_oob_selftest(); "
             "print('count', gc.debug_oob_count(), gc.version())")
    assert r.returncode == 0, r.stderr
    assert "count 1 " in r.stdout and "bounds-check" in r.stdout, r.stdout


def test_every_path_in_bounds(cuda_device):
    r = _run("import runpy, sys; sys.argv = ['sanitize_cases']; "
             "sys.exit(runpy.run_path('tools/sanitize_cases.py', run_name='__main__'))")
    assert r.returncode == 0, r.stdout + r.stderr
    assert "out-of-bounds accesses: 0" in r.stdout, r.stdout


def test_product_library_has_no_checks(cuda_device):
    import paper_1605_02178_b200 as gc
    if "bounds-check" in gc.version():
        pytest.skip("GC_LIB_PATH points at the check build")
    with pytest.raises(gc.GCError):
        gc.debug_oob_count()
