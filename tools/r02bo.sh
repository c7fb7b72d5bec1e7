#!/bin/bash
# column pass fold warps: f prefetched 3 (r_pf3) / 6 (s_pf6) blocks ahead with a running pointer, vs 1 block (q_base = HEAD)
O=gpurun_out/r02bo; mkdir -p $O
GC_LIB_PATH=$PWD/abl/r_pf3.so timeout 900 python -m pytest tests/test_gpu_operator.py -m gpu -x -q > $O/pytest_r.log 2>&1; echo "pytest r_pf3 rc=$?" >> $O/pytest.log
TAILN=5 bash tools/ab.sh r02bo "c5 --op 2" > /dev/null
TAILN=5 bash tools/ab.sh r02bo "c5 --op 2" > /dev/null
