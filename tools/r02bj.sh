#!/bin/bash
# column pass: y-segment count (GC_O1_COL_NSEG) — wave quantisation vs lead-in
O=gpurun_out/r02bj; mkdir -p $O
TAILN=1 bash tools/gpu_ab_env.sh r02bj "c5 --op 2" "GC_O1_COL_NSEG=0" "GC_O1_COL_NSEG=6" "GC_O1_COL_NSEG=12" "GC_O1_COL_NSEG=13" "GC_O1_COL_NSEG=16" > /dev/null
TAILN=3 bash tools/gpu_ab_env.sh r02bj "c3 --op 2 --sigma-s 10 20 40" "GC_O1_COL_NSEG=0" "GC_O1_COL_NSEG=7" "GC_O1_COL_NSEG=10" "GC_O1_COL_NSEG=14" > /dev/null
