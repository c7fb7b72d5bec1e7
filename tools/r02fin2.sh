set -u
# bench lines with hbm.dram_measured (bench.py after c0f0959), same library as r02fin
O=gpurun_out/r02fin2; mkdir -p $O
timeout 900 python bench.py > $O/bench_c5.json 2> $O/bench_c5.err; echo "bench c5 exit $?"
timeout 900 python bench.py --force-bands --steps 10 > $O/bench_c5_bands.json 2> $O/bench_c5_bands.err; echo "bench c5 bands exit $?"
timeout 600 python bench.py --workload c4 --steps 20 > $O/bench_c4.json 2> $O/bench_c4.err; echo "bench c4 exit $?"
timeout 600 python bench.py --workload c3 --sigma-s 40 --steps 50 --no-cpu-baseline > $O/bench_c3s40.json 2> $O/bench_c3s40.err; echo "bench c3 s40 exit $?"
