set -u
O=gpurun_out/r02n; mkdir -p $O
timeout 300 python tools/sanitize_cases.py > $O/plain.log 2>&1 && \
timeout 1500 compute-sanitizer --tool memcheck --leak-check full --print-limit 50 python tools/sanitize_cases.py > $O/memcheck.log 2>&1; echo "memcheck exit $?"; tail -5 $O/memcheck.log
