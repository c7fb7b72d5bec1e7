set -u
O=gpurun_out/$1; mkdir -p $O
python -m pytest tests/test_gpu_operator.py -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
tail -2 $O/pytest_gpu.log
timeout 300 python tools/time_ops.py c3 --sigma-s 2 5 10 20 40 --op 2 > $O/time_c3.txt 2>&1; cat $O/time_c3.txt
timeout 600 python tools/time_ops.py c5 --reps 5 --op 2 > $O/time_c5.txt 2>&1; cat $O/time_c5.txt
