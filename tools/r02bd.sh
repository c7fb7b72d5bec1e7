#!/bin/bash
# column pass on the running-pointer fold (d_run): fold slack 3 / 4 tile buffers (f_t3, g_t4), tile_free wait with nanosleep back-off (h_tfb); vs HEAD
O=gpurun_out/r02bd; mkdir -p $O
TAILN=5 bash tools/ab.sh r02bd "c5 --op 2" "c3 --op 2 --sigma-s 10 40" > /dev/null
