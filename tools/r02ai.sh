#!/bin/bash
# row pass: persistent dynamic tasks (LPT group order, balanced groups) vs static grid; NSEG sweep
O=gpurun_out/r02ai; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_operator.py tests/test_gpu_parity.py -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
TAILN=4 bash tools/ab.sh r02ai "c5" "c3 --op 2 --sigma-s 2 10 20 40" > /dev/null
bash tools/gpu_ab_env.sh r02ai "c5" "GC_O1_ROW_NSEG=5" "GC_O1_ROW_NSEG=8" "GC_O1_ROW_NSEG=12" "GC_O1_ROW_NSEG=16" "GC_O1_ROW_NSEG=24" "GC_O1_ROW_NSEG=32" > /dev/null
for n in 4 6 8 13 16 24; do TAILN=5 bash tools/gpu_ab_env.sh r02ai "c3 --op 2 --sigma-s 2 10 40" "GC_O1_ROW_NSEG=$n" > /dev/null; done
