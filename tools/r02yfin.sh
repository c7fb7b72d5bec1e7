set -u
# final evidence for the fold-prefetch build: full GPU suite, smoke, bands line, launch list with DRAM bytes
O=gpurun_out/r02yfin; mkdir -p $O
timeout 600 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -1 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?"; tail -1 $O/smoke.log
timeout 600 python bench.py --force-bands --steps 10 > $O/bench_c5_bands.json 2> $O/bench_c5_bands.err; echo "bench c5 bands exit $?"
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-sweep --no-check"
timeout 600 $CMD > $O/plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_c5.csv $CMD > $O/ncu_launch.log 2>&1; echo "ncu launch exit $?"
