#!/bin/bash
# row pass: two steps per loop iteration (register renaming of the Ep/Lp hand-over)
O=gpurun_out/r02ar; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_operator.py -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
TAILN=5 bash tools/ab.sh r02ar "c5 --op 2" "c3 --op 2 --sigma-s 2 10 20 40" > /dev/null
