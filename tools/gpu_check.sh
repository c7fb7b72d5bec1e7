#!/bin/bash
# Quick GPU check: gpu tests, smoke, default bench line.   usage: tools/gpu_check.sh <tag>
set -u
O=gpurun_out/${1:-check}; mkdir -p $O
python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log; tail -2 $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?"; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err; echo "bench c2 exit $?"; cat $O/bench_c2.json
