set -u
# evidence after the r02ax column-pass change: GPU tests, smoke, default bench line, launch list
O=gpurun_out/r02ay; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > $O/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo "pytest exit $?"; tail -1 $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?"; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench_c5.json 2> $O/bench_c5.err; echo "bench c5 exit $?"
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-sweep --no-check"
timeout 600 $CMD > $O/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_c5.csv $CMD > $O/ncu_launch.log 2>&1; echo "ncu launch exit $?"
