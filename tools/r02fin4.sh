set -u
# final evidence for the build with the fold-warp f prefetch: GPU tests, smoke, bench lines, launch list, ncu full
O=gpurun_out/r02fin4; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > $O/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo "pytest exit $?"; tail -1 $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?"; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench_c5.json 2> $O/bench_c5.err; echo "bench c5 exit $?"
timeout 900 python bench.py --force-bands --steps 10 > $O/bench_c5_bands.json 2> $O/bench_c5_bands.err; echo "bench c5 bands exit $?"
timeout 600 python bench.py --workload c3 --sigma-s 40 --steps 50 --no-cpu-baseline > $O/bench_c3s40.json 2> $O/bench_c3s40.err; echo "bench c3 s40 exit $?"
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-sweep --no-check"
timeout 600 $CMD > $O/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_c5.csv $CMD > $O/ncu_launch.log 2>&1; echo "ncu launch exit $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_(row|col)_o1" -s 2 -c 2 -o $O/o1_c5 python tools/time_ops.py c5 --op 2 --reps 1 > $O/ncu_full.log 2>&1; echo "ncu full exit $?"
