#!/bin/bash
# column pass: fold blocks of one ring stage (4 rows, fold rotating over the warps), 2 or 4 tile buffers
O=gpurun_out/r02ax; mkdir -p $O
for so in b_sb2 c_sb4; do
  GC_LIB_PATH=$PWD/abl/$so.so timeout 900 python -m pytest tests/test_gpu_operator.py tests/test_gpu_parity.py -m gpu -x -q > $O/pytest_$so.log 2>&1; echo "pytest $so rc=$?" >> $O/pytest.log
done
TAILN=5 bash tools/ab.sh r02ax "c5 --op 2" "c3 --op 2 --sigma-s 2 10 20 40" > /dev/null
