set -u
O=gpurun_out/$1; mkdir -p $O
CMD="python tools/time_ops.py c5 --H 4096 --W 4096 --op 2 --reps 1"
$CMD > $O/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:o1 -s 2 -c 2 -o $O/prof $CMD > $O/ncu_full.log 2>&1
echo "ncu exit $?"
