#!/bin/bash
# default bench.py three times with a Python stack dump after 400 s
O=gpurun_out/${TAG:-r02bp}; mkdir -p $O
for i in 1 2 3; do
  timeout 600 python -c "import faulthandler, sys, time; faulthandler.dump_traceback_later(400, exit=True); sys.argv=['bench.py']; t=time.time(); import runpy; runpy.run_path('bench.py', run_name='__main__'); print('elapsed', time.time()-t, file=sys.stderr)" > $O/bench_$i.json 2> $O/bench_$i.err
  echo "run $i exit $?"; tail -3 $O/bench_$i.err
  nvidia-smi --query-gpu=clocks.sm,power.draw,temperature.gpu --format=csv,noheader
done
