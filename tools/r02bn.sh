#!/bin/bash
# production build with fold warps for NP = 7: GPU tests (incl. bounds-check build), timing, bench
O=gpurun_out/r02bn; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo "pytest exit $?"; tail -1 $O/pytest.log
timeout 600 python tools/time_ops.py c5 --op 2 > $O/time_c5.txt 2>&1; tail -1 $O/time_c5.txt
timeout 900 python bench.py > $O/bench_c5.json 2> $O/bench_c5.err; echo "bench c5 exit $?"
