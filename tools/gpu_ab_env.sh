#!/bin/bash
# A/B of environment-selected kernel variants (development): tools/gpu_ab_env.sh <tag> "<time_ops args>" "ENV=.. ENV2=.." ...
set -u
O=gpurun_out/${1}; shift; mkdir -p $O
ARGS=$1; shift
for rep in 1 2; do
  for envs in "$@"; do
    echo -n "[$envs] "; env $envs timeout 300 python tools/time_ops.py $ARGS 2>&1 | tail -${TAILN:-1}
  done
done | tee -a $O/ab.txt
