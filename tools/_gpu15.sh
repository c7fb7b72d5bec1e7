set -u
for cfg in "0 0" "32 0" "0 120000" "32 120000" "32 80000"; do
set -- $cfg
echo "DBG=$1 COLSMEM=$2"
GC_DBG=$1 GC_COLSMEM=$2 timeout 300 python tools/time_ops.py c5 --op 2 --reps 3 2>&1 | tail -1
GC_DBG=$1 GC_COLSMEM=$2 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:k_col_o1 -s 2 -c 1 python tools/time_ops.py c5 --op 2 --reps 1 2>&1 | grep -E "dram|duration"
done
