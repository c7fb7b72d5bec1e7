set -u
O=gpurun_out/r02p; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_operator.py -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest exit $?"; tail -2 $O/pytest.log
TAILN=1 tools/gpu_ab_env.sh r02p "c5 --op 2 --reps 5" "GC_O1P_CTAS=3"
TAILN=5 tools/gpu_ab_env.sh r02p "c3 --op 2 --sigma-s 2 5 10 20 40 --reps 10" "GC_O1P_CTAS=3"
CMD="python tools/time_ops.py c5 --H 8192 --W 8192 --op 2 --reps 1"
timeout 300 $CMD > $O/plain.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_row_o1" -s 1 -c 1 -o $O/prof $CMD > $O/ncu.log 2>&1; echo "ncu exit $?"
