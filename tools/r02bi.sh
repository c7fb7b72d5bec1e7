#!/bin/bash
# row pass: recursion constants in ordinary registers (m_creg) vs uniform registers reloaded per step (l_c0 = HEAD)
O=gpurun_out/r02bi; mkdir -p $O
GC_LIB_PATH=$PWD/abl/m_creg.so timeout 900 python -m pytest tests/test_gpu_operator.py -m gpu -x -q > $O/pytest_m_creg.log 2>&1; echo "pytest m_creg rc=$?" >> $O/pytest.log
TAILN=5 bash tools/ab.sh r02bi "c5 --op 2" "c3 --op 2 --sigma-s 10 40" > /dev/null
