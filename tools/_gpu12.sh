for d in 0 8 16 24; do echo "GC_DBG=$d"; GC_DBG=$d timeout 300 python tools/time_ops.py c5 --H 8192 --W 8192 --op 2 --reps 5 2>&1 | tail -1; done
