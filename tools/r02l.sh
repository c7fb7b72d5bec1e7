set -u
O=gpurun_out/r02l; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_operator.py tests/test_gpu_parity.py -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest exit $?"; tail -3 $O/pytest.log
TAILN=1 tools/gpu_ab_env.sh r02l "c5 --op 2 --reps 5" "GC_O1P_CTAS=3" "GC_O1P_CTAS=2" "GC_O1_COL_LEGACY=1"
TAILN=5 tools/gpu_ab_env.sh r02l "c3 --op 2 --sigma-s 2 5 10 20 40 --reps 10" "GC_O1P_CTAS=3"
CMD="python tools/time_ops.py c5 --H 8192 --W 8192 --op 2 --reps 1"
timeout 300 $CMD > $O/plain.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_(row|col)_o1" -s 2 -c 2 -o $O/prof $CMD > $O/ncu.log 2>&1; echo "ncu exit $?"
