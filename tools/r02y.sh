set -u
O=gpurun_out/r02y; mkdir -p $O
GC_O1_COL_FLAT=1 timeout 900 python -m pytest tests/test_gpu_operator.py tests/test_gpu_parity.py -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest exit $?"; tail -3 $O/pytest.log
TAILN=1 tools/gpu_ab_env.sh r02y "c5 --op 2 --reps 5" "GC_O1_COL_FLAT=0" "GC_O1_COL_FLAT=1" "GC_O1_COL_FLAT=1 GC_O1P_CTAS=2"
TAILN=3 tools/gpu_ab_env.sh r02y "c3 --op 2 --sigma-s 2 10 40 --reps 10" "GC_O1_COL_FLAT=0" "GC_O1_COL_FLAT=1"
