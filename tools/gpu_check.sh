#!/bin/bash
# One GPU session: parity tests, benches, launch list and one full ncu capture.
# usage: tools/gpu_check.sh <tag> [kernel-regex] [workload]
set -u
TAG=${1:-run}; KRX=${2:-k_col}; WL=${3:-c2}
O=gpurun_out/$TAG; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err; echo "bench c2 exit $?"
timeout 600 python bench.py --workload c4 --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err; echo "bench c4 exit $?"
CMD="python bench.py --workload $WL --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > $O/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $CMD > $O/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$KRX -s 3 -c 1 -o $O/prof $CMD > $O/ncu_full.log 2>&1
echo "ncu exit $?"
