set -u
O=gpurun_out/r02aa; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_operator.py tests/test_gpu_parity.py -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest exit $?"; tail -2 $O/pytest.log
TAILN=1 tools/gpu_ab_env.sh r02aa "c5 --op 2 --reps 5" "X=1"
TAILN=8 tools/gpu_ab_env.sh r02aa "c3 --sigma-s 5 6 7 8 --reps 10" "X=1"
