set -u
O=gpurun_out/r02c; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_operator.py tests/test_gpu_parity.py -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest exit $?"; tail -3 $O/pytest.log
TAILN=1 tools/gpu_ab_env.sh r02c "c5 --op 2 --reps 5" "GC_O1_COL_LEGACY=1" "GC_O1P_CTAS=1" "GC_O1P_CTAS=2" "GC_O1P_CTAS=3" "GC_O1P_CTAS=2 GC_O1P_STAGES=16" "GC_O1P_CTAS=4"
TAILN=5 tools/gpu_ab_env.sh r02c "c3 --op 2 --sigma-s 2 10 40 --reps 10" "GC_O1_COL_LEGACY=1" "GC_O1P_CTAS=2" "GC_O1P_CTAS=3"
