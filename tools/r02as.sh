#!/bin/bash
# fused small-image FIR kernel: bit-exactness vs the two-pass path, oracle parity, timing, crossover
O=gpurun_out/r02as; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_parity.py tests/test_gpu_operator.py -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
for e in "GC_FIR_FUSED=1" "GC_FIR_FUSED=0"; do
  for c in "c1 --op 1" "c2 --op 1" "c4 --op 1 --B 4" "c3 --op 1 --sigma-s 2 5 8 --H 1024 --W 1024" "c3 --op 1 --sigma-s 2 5 8 --H 2048 --W 2048" "c3 --op 1 --sigma-s 2 5 8"; do
    TAILN=3 bash tools/gpu_ab_env.sh r02as "$c --reps 50" "$e" > /dev/null
  done
done
timeout 600 python bench.py --workload c1 --steps 200 > $O/bench_c1.json 2> $O/bench_c1.err; echo "bench c1 exit $?" >> $O/pytest.log
timeout 600 python bench.py --workload c2 --steps 200 > $O/bench_c2.json 2> $O/bench_c2.err; echo "bench c2 exit $?" >> $O/pytest.log
