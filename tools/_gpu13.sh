set -u
O=gpurun_out/$1; mkdir -p $O
CMD="python tools/time_ops.py c5 --op 2 --reps 1"
$CMD > $O/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:o1 -s 2 -c 2 $CMD > $O/ncu.txt 2>&1
echo "ncu exit $?"; grep -E "k_|dram|time|hit|fma|issue" $O/ncu.txt | head -20
