set -u
O=gpurun_out/$1; mkdir -p $O
for cfg in "4 100000" "4 70000" "8 100000" "8 70000" "2 100000"; do
set -- $cfg
echo "G=$1 smem=$2"
GC_COLG=$1 GC_COLSMEM=$2 timeout 300 python tools/time_ops.py c5 --op 2 --reps 3 2>&1 | tail -1
done
