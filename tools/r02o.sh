set -u
O=gpurun_out/r02o; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_bounds.py -m gpu -q -x > $O/pytest_bounds.log 2>&1; echo "bounds pytest exit $?"; tail -5 $O/pytest_bounds.log
GC_LIB_PATH=$PWD/paper_1605_02178_b200/libgc_check.so timeout 600 python tools/sanitize_cases.py > $O/sanitize_cases.log 2>&1; echo "cases exit $?"; tail -2 $O/sanitize_cases.log
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -2 $O/pytest_gpu.log
