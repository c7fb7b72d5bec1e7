#!/bin/bash
# direct lead-in in the pair-parallel column pass too; row NSEG rule
O=gpurun_out/r02al; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
TAILN=5 bash tools/gpu_ab_env.sh r02al "c3 --op 2 --sigma-s 2 5 10 20 40" "GC_O1_DIRECT_LEAD=1" "GC_O1_DIRECT_LEAD=0" > /dev/null
bash tools/gpu_ab_env.sh r02al "c5 --op 2" "GC_O1_DIRECT_LEAD=1" "GC_O1_DIRECT_LEAD=0" > /dev/null
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
