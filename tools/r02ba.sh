#!/bin/bash
# per-SMSP balance of the column pass (max / min / avg over the GPU's SMSPs)
O=gpurun_out/r02ba; mkdir -p $O
M=smsp__inst_executed.sum,smsp__inst_executed.max,smsp__inst_executed.min,smsp__inst_executed.avg,smsp__pipe_fma_cycles_active.max,smsp__pipe_fma_cycles_active.min,smsp__pipe_fma_cycles_active.avg,smsp__issue_active.max,smsp__issue_active.min,smsp__issue_active.avg,smsp__warps_launched.max,smsp__warps_launched.min,smsp__warps_launched.avg,sm__cycles_elapsed.avg,smsp__cycles_active.avg,smsp__cycles_active.min,smsp__cycles_active.max
python tools/time_ops.py c3 --op 2 --sigma-s 10 --reps 2 > $O/plain.txt 2>&1 && \
timeout 600 ncu --metrics $M --clock-control none -k regex:"k_(row|col)_o1" -c 4 --csv python tools/time_ops.py c3 --op 2 --sigma-s 10 --reps 1 > $O/smsp_c3.csv 2> $O/ncu.err
echo "ncu exit $?"
timeout 600 ncu --metrics $M --clock-control none -k regex:"k_(row|col)_o1" -c 2 --csv python tools/time_ops.py c5 --op 2 --reps 1 > $O/smsp_c5.csv 2>> $O/ncu.err
echo "ncu c5 exit $?"
