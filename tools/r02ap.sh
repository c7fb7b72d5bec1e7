#!/bin/bash
# row pass task order: group-major (LPT) vs group-minor (f shared in L2)
O=gpurun_out/r02ap; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_operator.py -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
bash tools/gpu_ab_env.sh r02ap "c5 --op 2" "GC_O1_ROW_ORDER=0" "GC_O1_ROW_ORDER=1" > /dev/null
TAILN=5 bash tools/gpu_ab_env.sh r02ap "c3 --op 2 --sigma-s 2 10 20 40" "GC_O1_ROW_ORDER=0" "GC_O1_ROW_ORDER=1" > /dev/null
