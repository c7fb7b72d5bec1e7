#!/bin/bash
# column pass: running fold rows / f and output pointers (d_run) vs HEAD (a_base)
O=gpurun_out/r02bb; mkdir -p $O
GC_LIB_PATH=$PWD/abl/d_run.so timeout 900 python -m pytest tests/test_gpu_operator.py tests/test_gpu_parity.py tests/test_gpu_bounds.py -m gpu -x -q > $O/pytest_d_run.log 2>&1; echo "pytest d_run rc=$?" >> $O/pytest.log
TAILN=5 bash tools/ab.sh r02bb "c5 --op 2" "c3 --op 2 --sigma-s 2 10 20 40" > /dev/null
