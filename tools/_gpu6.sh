set -u
O=gpurun_out/$1; mkdir -p $O
python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
timeout 600 python bench.py --steps 100 --no-e2e --no-cpu-baseline > $O/bench_c2.json 2> $O/bench_c2.err; echo "bench c2 exit $?"; python -c "
import json; d=json.load(open('$O/bench_c2.json')); print('c2', d['value'], d['ms_per_step'], d['kernels'])"
timeout 600 python bench.py --workload c4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_c4.json 2> $O/bench_c4.err; echo "bench c4 exit $?"; python -c "
import json; d=json.load(open('$O/bench_c4.json')); print('c4', d['value'], d['ms_per_step'], d['kernels'])"
timeout 300 python tools/time_ops.py c3 --sigma-s 2 5 --op 1 > $O/time_c3.txt 2>&1; cat $O/time_c3.txt
