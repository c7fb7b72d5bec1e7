set -u
O=gpurun_out/r02ab; mkdir -p $O
GC_LIB_PATH=$PWD/abl/b_hints.so timeout 900 python -m pytest tests/test_gpu_operator.py -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest exit $?"; tail -2 $O/pytest.log
TAILN=1 tools/ab.sh r02ab "c5 --op 2 --reps 5"
TAILN=3 tools/ab.sh r02ab "c3 --op 2 --sigma-s 2 10 40 --reps 10"
for so in a_nohint b_hints; do GC_LIB_PATH=$PWD/abl/$so.so timeout 300 python tools/time_ops.py c5 --op 2 --reps 1 > /dev/null 2>&1 && GC_LIB_PATH=$PWD/abl/$so.so timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none --csv --log-file $O/dram_$so.csv python tools/time_ops.py c5 --op 2 --reps 1 > /dev/null 2>&1; echo "ncu $so exit $?"; done
