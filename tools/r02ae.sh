set -u
O=gpurun_out/r02ae; mkdir -p $O
run() { timeout 600 python bench.py --steps 40 --warmup 5 --no-e2e --no-cpu-baseline --no-sweep --no-check 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']), round(d['ms_per_step'],3), d['clocks'], d['kernels']['k_row']['ms'], d['kernels']['k_col']['ms'])"; }
for rep in 1 2; do
  echo -n "base: "; GC_LIB_PATH=$PWD/abl/a_base.so run
  echo -n "sleep: "; GC_LIB_PATH=$PWD/abl/b_sleep.so run
  echo -n "base CTAS=2: "; GC_O1P_CTAS=2 GC_LIB_PATH=$PWD/abl/a_base.so run
done | tee $O/power.txt
