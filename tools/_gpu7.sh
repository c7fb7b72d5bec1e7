set -u
O=gpurun_out/$1; mkdir -p $O
python -m pytest tests/test_gpu_direct.py -x -q > $O/pytest_direct.log 2>&1; echo "pytest exit $?" >> $O/pytest_direct.log; tail -3 $O/pytest_direct.log
timeout 300 python tools/c1_graph.py > $O/c1_graph.txt 2>&1; cat $O/c1_graph.txt
timeout 1500 python tools/quality.py > $O/quality.md 2> $O/quality.err; echo "quality exit $?"; cat $O/quality.md; tail -5 $O/quality.err
