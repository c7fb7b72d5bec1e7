#!/bin/bash
# column pass y-segment count sweep (static grid)
O=gpurun_out/r02am; mkdir -p $O
bash tools/gpu_ab_env.sh r02am "c5 --op 2" "GC_O1_COL_NSEG=0" "GC_O1_COL_NSEG=3" "GC_O1_COL_NSEG=4" "GC_O1_COL_NSEG=5" "GC_O1_COL_NSEG=8" "GC_O1_COL_NSEG=12" "GC_O1_COL_NSEG=16" > /dev/null
for n in 0 2 3 4 6 8 10 16; do TAILN=5 bash tools/gpu_ab_env.sh r02am "c3 --op 2 --sigma-s 2 10 20 40" "GC_O1_COL_NSEG=$n" > /dev/null; done
