#!/bin/bash
# column y-segment rule: parity + timing
O=gpurun_out/r02an; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_operator.py tests/test_gpu_parity.py -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
TAILN=5 bash tools/gpu_ab_env.sh r02an "c3 --op 2 --sigma-s 2 5 10 20 40" "X=1" > /dev/null
bash tools/gpu_ab_env.sh r02an "c5 --op 2" "X=1" > /dev/null
