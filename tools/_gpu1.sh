set -u
O=gpurun_out/r01b; mkdir -p $O
python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
timeout 300 python tools/time_ops.py c3 --sigma-s 2 5 10 20 40 > $O/time_c3.txt 2>&1; cat $O/time_c3.txt
timeout 300 python tools/time_ops.py c2 > $O/time_c2.txt 2>&1; cat $O/time_c2.txt
timeout 300 python tools/time_ops.py c4 --B 64 > $O/time_c4.txt 2>&1; cat $O/time_c4.txt
timeout 600 python tools/time_ops.py c5 --reps 5 > $O/time_c5.txt 2>&1; cat $O/time_c5.txt
