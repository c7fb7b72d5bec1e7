#!/bin/bash
# direct lead-in of the row pass: parity + A/B against the recursion lead-in
O=gpurun_out/r02af; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
for c in "c5" "c3 --op 2 --sigma-s 2 10 20 40"; do
  bash tools/gpu_ab_env.sh r02af "$c" "GC_O1_DIRECT_LEAD=1" "GC_O1_DIRECT_LEAD=0" > /dev/null
done
TAILN=5 bash tools/gpu_ab_env.sh r02af "c3 --op 2 --sigma-s 2 10 20 40" "GC_O1_DIRECT_LEAD=1" > /dev/null
