set -u
O=gpurun_out/r02ad; mkdir -p $O
for rep in 1 2; do
for v in a_trig_start c_trig_end; do
  echo -n "$v: "; GC_LIB_PATH=$PWD/abl/$v.so timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-sweep --no-check 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']), round(d['ms_per_step'],3), d['clocks'])"
  echo -n "$v NO_PDL: "; GC_NO_PDL=1 GC_LIB_PATH=$PWD/abl/$v.so timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-sweep --no-check 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']), round(d['ms_per_step'],3), d['clocks'])"
done; done | tee $O/pdl.txt
