set -u
O=gpurun_out/$1; mkdir -p $O
CMD="python bench.py --workload c2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > $O/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_(row|col)_t" -s 6 -c 2 -o $O/prof $CMD > $O/ncu_full.log 2>&1
echo "ncu exit $?"
