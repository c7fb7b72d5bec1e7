set -u
O=gpurun_out/r02r; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 $O/pytest_gpu.log
TAILN=1 tools/gpu_ab_env.sh r02r "c5 --op 2 --reps 5" "GC_O1P_CTAS=3" "GC_O1P_CTAS=2"
TAILN=5 tools/gpu_ab_env.sh r02r "c3 --op 2 --sigma-s 2 5 10 20 40 --reps 10" "GC_O1P_CTAS=3"
timeout 900 python bench.py > $O/bench_c5.json 2> $O/bench_c5.err; echo "bench c5 exit $?"; tail -c 600 $O/bench_c5.json
