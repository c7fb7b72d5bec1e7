#!/bin/bash
# column pass: 4 dedicated fold warps, consumers only filter, 2 CTAs/SM (n_fold4) vs production (o_base)
O=gpurun_out/r02bl; mkdir -p $O
GC_LIB_PATH=$PWD/abl/n_fold4.so timeout 900 python -m pytest tests/test_gpu_operator.py tests/test_gpu_parity.py -m gpu -x -q > $O/pytest_n_fold4.log 2>&1; echo "pytest n_fold4 rc=$?" >> $O/pytest.log
TAILN=5 bash tools/ab.sh r02bl "c5 --op 2" "c3 --op 2 --sigma-s 10 40" > /dev/null
GC_LIB_PATH=$PWD/abl/n_fold4.so timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_col_o1p -c 1 --csv python tools/time_ops.py c5 --op 2 --reps 1 > $O/ncu_n_fold4.csv 2>&1; echo "ncu rc=$?"
