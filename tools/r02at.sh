#!/bin/bash
# fused small-image FIR kernel: tests, crossover sizes, bench c1, ncu of the fused kernel at c2
O=gpurun_out/r02at; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_abi.py -m "gpu or not gpu" -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
for e in "GC_FIR_FUSED=1" "GC_FIR_FUSED=0"; do
  for hw in 256 384 512 768; do
    TAILN=1 bash tools/gpu_ab_env.sh r02at "c1 --op 1 --reps 50 --H $hw --W $hw" "$e" > /dev/null
    TAILN=1 bash tools/gpu_ab_env.sh r02at "c2 --op 1 --reps 50 --H $hw --W $hw" "$e" > /dev/null
  done
done
timeout 600 python bench.py --workload c1 --steps 200 > $O/bench_c1.json 2> $O/bench_c1.err; echo "bench c1 exit $?" >> $O/pytest.log
CMD="python tools/time_ops.py c2 --op 1 --reps 2"
GC_FIR_FUSED=1 timeout 300 $CMD > $O/plain.log 2>&1 && GC_FIR_FUSED=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_fused" -s 3 -c 1 -o $O/prof_fused $CMD > $O/ncu.log 2>&1; echo "ncu exit $?" >> $O/pytest.log
