#!/bin/bash
# Round evidence on one B200: tests, smoke, bench lines (c2 default, c4, c5, Deriche mode),
# the c3 sigma_s sweep, c1 CUDA-graph timing, the launch list of the default bench and one
# ncu --set full capture of its dominant kernels.   usage: tools/gpu_round.sh <tag>
set -u
O=gpurun_out/${1:-round}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log; tail -2 $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?"; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err; echo "bench c2 exit $?"
timeout 900 python bench.py --workload c4 --steps 20 --warmup 3 > $O/bench_c4.json 2> $O/bench_c4.err; echo "bench c4 exit $?"
timeout 900 python bench.py --workload c5 --steps 10 --warmup 3 > $O/bench_c5.json 2> $O/bench_c5.err; echo "bench c5 exit $?"
timeout 900 python bench.py --workload c1 --steps 200 --warmup 5 > $O/bench_c1.json 2> $O/bench_c1.err; echo "bench c1 exit $?"
timeout 900 python bench.py --op 3 --no-e2e --no-cpu-baseline > $O/bench_c2_deriche.json 2> $O/bench_c2_deriche.err; echo "bench c2 deriche exit $?"
timeout 900 python bench.py --workload c5 --op 3 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_c5_deriche.json 2> $O/bench_c5_deriche.err; echo "bench c5 deriche exit $?"
timeout 900 python tools/time_ops.py c3 --sigma-s 2 5 10 20 40 > $O/time_c3.txt 2>&1
timeout 600 python tools/c1_graph.py > $O/c1_graph.txt 2>&1
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > $O/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $CMD > $O/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_(row|col)_t" -s 6 -c 2 -o $O/prof $CMD > $O/ncu_full.log 2>&1
echo "ncu exit $?"
