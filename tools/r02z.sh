set -u
O=gpurun_out/r02z; mkdir -p $O
GC_LIB_PATH=$PWD/abl/b_staged.so timeout 900 python -m pytest tests/test_gpu_operator.py -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest exit $?"; tail -2 $O/pytest.log
TAILN=1 tools/ab.sh r02z "c5 --op 2 --reps 5"
TAILN=3 tools/ab.sh r02z "c3 --op 2 --sigma-s 2 10 40 --reps 10"
