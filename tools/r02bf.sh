#!/bin/bash
# ncu --set full of both O(1) kernels at c5 (production build after r02be), source-level stalls
O=gpurun_out/r02bf; mkdir -p $O
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_(row|col)_o1" -s 2 -c 2 -o $O/o1_c5 python tools/time_ops.py c5 --op 2 --reps 1 > $O/ncu.log 2>&1; echo "ncu exit $?"
