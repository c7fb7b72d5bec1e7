set -u
O=gpurun_out/r02m; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?"; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench_c5.json 2> $O/bench_c5.err; echo "bench c5 exit $?"
timeout 600 python bench.py --workload c2 --steps 200 --no-sweep > $O/bench_c2.json 2> $O/bench_c2.err; echo "bench c2 exit $?"
timeout 600 python bench.py --workload c4 --steps 20 --no-sweep > $O/bench_c4.json 2> $O/bench_c4.err; echo "bench c4 exit $?"
for so in abl/*.so; do for r in 1 2; do echo -n "$(basename $so) | "; GC_LIB_PATH=$PWD/$so timeout 300 python tools/time_ops.py c5 --op 2 --reps 5 2>&1 | tail -1; done; done | tee $O/ab_rowinline.txt
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-sweep --no-check"
timeout 600 $CMD > $O/plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches.csv $CMD > $O/ncu_launch.log 2>&1; echo "ncu launch exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_(row|col)_o1" -s 6 -c 2 -o $O/prof $CMD > $O/ncu_full.log 2>&1; echo "ncu full exit $?"
