#!/bin/bash
# row pass NSEG sweep with the dynamic fetch
O=gpurun_out/r02ak; mkdir -p $O
bash tools/gpu_ab_env.sh r02ak "c5 --op 2" "GC_O1_ROW_NSEG=7" "GC_O1_ROW_NSEG=9" "GC_O1_ROW_NSEG=12" "GC_O1_ROW_NSEG=16" "GC_O1_ROW_NSEG=24" > /dev/null
for n in 24 32 48; do TAILN=5 bash tools/gpu_ab_env.sh r02ak "c3 --op 2 --sigma-s 2 10 40" "GC_O1_ROW_NSEG=$n" > /dev/null; done
for n in 2 4 8 16; do TAILN=5 bash tools/gpu_ab_env.sh r02ak "c3 --op 2 --sigma-s 10 --H 2048 --W 2048 --B 1" "GC_O1_ROW_NSEG=$n" > /dev/null; done
