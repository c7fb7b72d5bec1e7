set -u
# ncu --set full of the O(1) pair in the default bench step (current kernels)
O=gpurun_out/r02aq; mkdir -p $O
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-sweep --no-check"
timeout 600 $CMD > $O/plain.log 2>&1; echo "plain exit $?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_(row_o1|col_o1p)" -s 6 -c 2 -o $O/prof_c5 $CMD > $O/ncu_full.log 2>&1; echo "ncu full c5 exit $?"
