O=gpurun_out/r02ac
mkdir -p $O
timeout 900 python bench.py --config c4 > $O/bench_c4.log 2>&1
timeout 900 python bench.py --config c4potts > $O/bench_c4potts.log 2>&1
tail -c 700 $O/bench_c4.log; tail -c 700 $O/bench_c4potts.log
