#!/bin/bash
# column pass: 4 dedicated fold warps at 3 CTAs/SM (56 registers, p_fold4c3) vs production (o_base)
O=gpurun_out/r02bm; mkdir -p $O
GC_LIB_PATH=$PWD/abl/p_fold4c3.so timeout 900 python -m pytest tests/test_gpu_operator.py -m gpu -x -q > $O/pytest_p.log 2>&1; echo "pytest p_fold4c3 rc=$?" >> $O/pytest.log
TAILN=5 bash tools/ab.sh r02bm "c5 --op 2" "c3 --op 2 --sigma-s 10 40" > /dev/null
