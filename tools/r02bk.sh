#!/bin/bash
# bench line with hbm.dram_measured (after the final evidence), and the band path's stdout hygiene
O=gpurun_out/r02bk; mkdir -p $O
timeout 900 python bench.py > $O/bench_c5.json 2> $O/bench_c5.err; echo "bench c5 exit $?"
timeout 900 python bench.py --force-bands --steps 10 --no-sweep --no-cpu-baseline > $O/bench_c5_bands.json 2> $O/bench_c5_bands.err; echo "bench bands exit $?"
wc -l $O/bench_c5.json $O/bench_c5_bands.json
