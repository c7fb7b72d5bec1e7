set -u
O=gpurun_out/r02ac; mkdir -p $O
GC_LIB_PATH=$PWD/abl/b_uniform.so timeout 900 python -m pytest tests/test_gpu_operator.py tests/test_gpu_parity.py -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest exit $?"; tail -2 $O/pytest.log
TAILN=1 tools/ab.sh r02ac "c5 --op 2 --reps 5"
TAILN=5 tools/ab.sh r02ac "c3 --op 2 --sigma-s 2 5 10 20 40 --reps 10"
