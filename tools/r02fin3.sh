set -u
# final evidence for build eefae37 (fold warps for NP = 7): smoke, c5 bench lines, launch list, ncu full of the O(1) pair
O=gpurun_out/r02fin3; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > $O/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?"; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench_c5.json 2> $O/bench_c5.err; echo "bench c5 exit $?"
timeout 900 python bench.py --force-bands --steps 10 > $O/bench_c5_bands.json 2> $O/bench_c5_bands.err; echo "bench c5 bands exit $?"
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-sweep --no-check"
timeout 600 $CMD > $O/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_c5.csv $CMD > $O/ncu_launch.log 2>&1; echo "ncu launch exit $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_(row|col)_o1" -s 2 -c 2 -o $O/o1_c5 python tools/time_ops.py c5 --op 2 --reps 1 > $O/ncu_full.log 2>&1; echo "ncu full exit $?"
