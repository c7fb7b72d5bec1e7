set -u
O=gpurun_out/$1; mkdir -p $O
python -m pytest tests/test_gpu_operator.py tests/test_gpu_parity.py -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
timeout 300 python tools/time_ops.py c3 --sigma-s 2 5 10 20 40 --op 2 > $O/time_c3.txt 2>&1; cat $O/time_c3.txt
timeout 600 python tools/time_ops.py c5 --reps 5 --op 2 > $O/time_c5.txt 2>&1; cat $O/time_c5.txt
CMD="python tools/time_ops.py c3 --sigma-s 5 --op 2 --reps 1"
$CMD > $O/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:o1 -s 2 -c 2 -o $O/prof $CMD > $O/ncu_full.log 2>&1
echo "ncu exit $?"
