#!/bin/bash
# row pass: unrolled direct lead-in; x-segment count sweep
O=gpurun_out/r02ag; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_operator.py tests/test_gpu_parity.py -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
bash tools/gpu_ab_env.sh r02ag "c5" "GC_O1_DIRECT_LEAD=1" "GC_O1_DIRECT_LEAD=0" "GC_O1_ROW_NSEG=2" "GC_O1_ROW_NSEG=3" "GC_O1_ROW_NSEG=4" "GC_O1_ROW_NSEG=6" "GC_O1_ROW_NSEG=8" > /dev/null
TAILN=5 bash tools/gpu_ab_env.sh r02ag "c3 --op 2 --sigma-s 2 10 20 40" "GC_O1_DIRECT_LEAD=1" "GC_O1_DIRECT_LEAD=0" > /dev/null
for n in 3 4 5 8 10 12; do TAILN=5 bash tools/gpu_ab_env.sh r02ag "c3 --op 2 --sigma-s 2 40" "GC_O1_ROW_NSEG=$n" > /dev/null; done
