set -u
O=gpurun_out/$1; mkdir -p $O
python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err; echo "bench c2 exit $?"; cat $O/bench_c2.json
timeout 600 python bench.py --workload c4 --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err; echo "bench c4 exit $?"; cat $O/bench_c4.json
timeout 900 python bench.py --workload c5 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_c5.json 2> $O/bench_c5.err; echo "bench c5 exit $?"; cat $O/bench_c5.json
