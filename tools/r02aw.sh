#!/bin/bash
# column pass: 3 fold tile buffers (2 ring stages at 3 CTAs/SM) vs 2 buffers (3 stages)
O=gpurun_out/r02aw; mkdir -p $O
GC_LIB_PATH=$PWD/abl/b_t3.so timeout 900 python -m pytest tests/test_gpu_operator.py -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
TAILN=5 bash tools/ab.sh r02aw "c5 --op 2" "c3 --op 2 --sigma-s 2 10 20 40" > /dev/null
