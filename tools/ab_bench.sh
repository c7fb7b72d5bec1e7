#!/bin/bash
# A/B of library builds in abl/*.so through bench.py (production call, PDL active) and time_ops.
O=gpurun_out/ab; mkdir -p $O
for rep in 1 2; do
  for so in abl/*.so; do
    v=$(GC_LIB_PATH=$PWD/$so timeout 300 python bench.py --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1000,1),'us', 'row', round(d['kernels']['k_row']['ms']*1000,1), 'col', round(d['kernels']['k_col']['ms']*1000,1))")
    echo "$(basename $so) c2 bench: $v"
  done
done | tee $O/ab_bench.txt
for args in "$@"; do
  for so in abl/*.so; do
    echo -n "$(basename $so) | "; GC_LIB_PATH=$PWD/$so python tools/time_ops.py $args 2>&1 | tail -1
  done
done | tee -a $O/ab_bench.txt
