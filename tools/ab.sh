#!/bin/bash
# A/B timing of library builds in abl/*.so (development tool): each variant twice, interleaved.
#   usage: tools/ab.sh "<time_ops args>" ["<time_ops args>" ...]
O=gpurun_out/ab; mkdir -p $O
for args in "$@"; do
  for rep in 1 2; do
    for so in abl/*.so; do
      echo -n "$(basename $so) | "; GC_LIB_PATH=$PWD/$so python tools/time_ops.py $args 2>&1 | tail -1
    done
  done
done | tee $O/ab.txt
