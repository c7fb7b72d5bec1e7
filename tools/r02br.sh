#!/bin/bash
# fold warps with the tile_free early-arrival fix: GPU tests, default bench twice (stack dump after 400 s)
O=gpurun_out/r02br; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo "pytest exit $?"; tail -1 $O/pytest.log
for i in 1 2; do
  timeout 600 python -c "import faulthandler, sys, runpy; faulthandler.dump_traceback_later(400, exit=True); sys.argv=['bench.py']; runpy.run_path('bench.py', run_name='__main__')" > $O/bench_$i.json 2> $O/bench_$i.err
  echo "bench $i exit $?"; tail -2 $O/bench_$i.err
done
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?"; tail -1 $O/smoke.log
