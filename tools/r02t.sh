set -u
O=gpurun_out/r02t; mkdir -p $O
timeout 900 python bench.py --force-bands --steps 5 --warmup 3 --no-sweep --no-cpu-baseline > $O/bench_bands1.json 2> $O/bench_bands1.err; echo "bench force-bands exit $?"; tail -c 1500 $O/bench_bands1.json; tail -3 $O/bench_bands1.err
CMD="python tools/time_ops.py c5 --H 8192 --W 8192 --op 2 --reps 1"
timeout 300 $CMD > $O/plain.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_(row|col)_o1" -s 2 -c 2 -o $O/prof $CMD > $O/ncu.log 2>&1; echo "ncu exit $?"
