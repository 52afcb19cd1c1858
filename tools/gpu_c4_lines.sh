mkdir -p gpurun_out/c4f
for c in c4 c4potts; do timeout 900 python bench.py --config $c > gpurun_out/c4f/bench_$c.log 2>&1; echo "$c rc=$?"; done
