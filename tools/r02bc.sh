#!/bin/bash
# column pass: running pointers with (e_run_wait) / without (d_run) the tile_full wait of non-folding warps, vs HEAD;
# ncu --set full of d_run's column pass at c5 (source-level stalls)
O=gpurun_out/r02bc; mkdir -p $O
TAILN=5 bash tools/ab.sh r02bc "c5 --op 2" "c3 --op 2 --sigma-s 2 10 40" > /dev/null
GC_LIB_PATH=$PWD/abl/d_run.so timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_col_o1p -s 1 -c 1 -o $O/colp_c5 python tools/time_ops.py c5 --op 2 --reps 1 > $O/ncu.log 2>&1; echo "ncu exit $?"
