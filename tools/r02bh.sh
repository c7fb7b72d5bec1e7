#!/bin/bash
# column pass: rolling tile-buffer / phase counters (j_roll), + fold lag of 2 blocks (k_lag2), vs i_bar0
O=gpurun_out/r02bh; mkdir -p $O
for so in j_roll k_lag2; do
GC_LIB_PATH=$PWD/abl/$so.so timeout 900 python -m pytest tests/test_gpu_operator.py -m gpu -x -q > $O/pytest_$so.log 2>&1; echo "pytest $so rc=$?" >> $O/pytest.log
done
TAILN=5 bash tools/ab.sh r02bh "c5 --op 2" "c3 --op 2 --sigma-s 10 40" > /dev/null
