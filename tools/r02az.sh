#!/bin/bash
# column pass: f of the fold loaded two blocks ahead (b_pf), + producer back-off 1000 ns (c_pf_ns1k), vs HEAD (a_base)
O=gpurun_out/r02az; mkdir -p $O
for so in b_pf; do
  GC_LIB_PATH=$PWD/abl/$so.so timeout 900 python -m pytest tests/test_gpu_operator.py tests/test_gpu_parity.py -m gpu -x -q > $O/pytest_$so.log 2>&1; echo "pytest $so rc=$?" >> $O/pytest.log
done
TAILN=5 bash tools/ab.sh r02az "c5 --op 2" "c3 --op 2 --sigma-s 2 10 20 40" > /dev/null
