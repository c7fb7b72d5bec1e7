set -u
O=gpurun_out/$1; mkdir -p $O
python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
timeout 600 python bench.py --steps 100 --no-cpu-baseline > $O/bench_c2.json 2> $O/bench_c2.err; echo "bench c2 exit $?"; python -c "
import json; d=json.load(open('$O/bench_c2.json')); print('c2', d['value'], d['e2e'])"
timeout 600 python bench.py --workload c4 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err; echo "bench c4 exit $?"; python -c "
import json; d=json.load(open('$O/bench_c4.json')); print('c4', d['value'], d['e2e'])"
