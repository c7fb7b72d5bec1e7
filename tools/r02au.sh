#!/bin/bash
# fused kernel v2 (batched staging loads, 4-wide row items on short tiles): tests + timing
O=gpurun_out/r02au; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_abi.py tests/test_gpu_parity.py -m "gpu or not gpu" -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
for e in "GC_FIR_FUSED=1" "GC_FIR_FUSED=0"; do
  for hw in 256 512 768; do
    TAILN=1 bash tools/gpu_ab_env.sh r02au "c1 --op 1 --reps 50 --H $hw --W $hw" "$e" > /dev/null
    TAILN=1 bash tools/gpu_ab_env.sh r02au "c2 --op 1 --reps 50 --H $hw --W $hw" "$e" > /dev/null
  done
done
timeout 600 python bench.py --workload c1 --steps 200 > $O/bench_c1.json 2> $O/bench_c1.err; echo "bench c1 exit $?" >> $O/pytest.log
timeout 600 python bench.py --workload c2 --steps 200 > $O/bench_c2.json 2> $O/bench_c2.err; echo "bench c2 exit $?" >> $O/pytest.log
