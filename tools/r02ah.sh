#!/bin/bash
# row pass x-segment count sweep at c5 and c3
O=gpurun_out/r02ah; mkdir -p $O
bash tools/gpu_ab_env.sh r02ah "c5" "GC_O1_ROW_NSEG=5" "GC_O1_ROW_NSEG=7" "GC_O1_ROW_NSEG=8" "GC_O1_ROW_NSEG=9" "GC_O1_ROW_NSEG=10" "GC_O1_ROW_NSEG=12" "GC_O1_ROW_NSEG=14" "GC_O1_ROW_NSEG=16" "GC_O1_ROW_NSEG=20" "GC_O1_ROW_NSEG=24" "GC_O1_ROW_NSEG=32" > /dev/null
for n in 6 7 13 14 16 20; do TAILN=5 bash tools/gpu_ab_env.sh r02ah "c3 --op 2 --sigma-s 2 10 40" "GC_O1_ROW_NSEG=$n" > /dev/null; done
