#!/bin/bash
# row pass: persistent dynamic tasks (LPT order, 4-pair groups) vs static grid; NSEG check
O=gpurun_out/r02aj; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_operator.py tests/test_gpu_parity.py -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
TAILN=4 bash tools/ab.sh r02aj "c5 --op 2" "c3 --op 2 --sigma-s 2 5 10 20 40" > /dev/null
bash tools/gpu_ab_env.sh r02aj "c5 --op 2" "GC_O1_ROW_NSEG=4" "GC_O1_ROW_NSEG=5" "GC_O1_ROW_NSEG=6" "GC_O1_ROW_NSEG=8" "GC_O1_ROW_NSEG=10" > /dev/null
for n in 6 8 12 16 20; do TAILN=5 bash tools/gpu_ab_env.sh r02aj "c3 --op 2 --sigma-s 2 10 40" "GC_O1_ROW_NSEG=$n" > /dev/null; done
