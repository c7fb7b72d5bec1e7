#!/bin/bash
# A/B timing of library builds in abl/*.so (development tool): each variant twice, interleaved.
#   usage: tools/ab.sh <tag> "<time_ops args>" ["<time_ops args>" ...]      (TAILN lines of output each)
O=gpurun_out/${1}; shift; mkdir -p $O
for args in "$@"; do
  for rep in 1 2; do
    for so in abl/*.so; do
      echo -n "$(basename $so) | "; GC_LIB_PATH=$PWD/$so timeout 300 python tools/time_ops.py $args 2>&1 | tail -${TAILN:-1}
    done
  done
done | tee -a $O/ab.txt
