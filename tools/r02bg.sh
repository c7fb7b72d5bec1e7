#!/bin/bash
# column pass: barrier block address kept in a register (i_bar0) vs HEAD; and 2 vs 3 column CTAs per SM on i_bar0
O=gpurun_out/r02bg; mkdir -p $O
GC_LIB_PATH=$PWD/abl/i_bar0.so timeout 900 python -m pytest tests/test_gpu_operator.py -m gpu -x -q > $O/pytest_i_bar0.log 2>&1; echo "pytest i_bar0 rc=$?" >> $O/pytest.log
TAILN=5 bash tools/ab.sh r02bg "c5 --op 2" "c3 --op 2 --sigma-s 10 40" > /dev/null
GC_LIB_PATH=$PWD/abl/i_bar0.so TAILN=5 bash tools/gpu_ab_env.sh r02bg "c5 --op 2" "GC_O1P_CTAS=3" "GC_O1P_CTAS=2" > /dev/null
