mkdir -p gpurun_out
for rep in 1 2; do
  python bench.py --config c2 --no-cpu-baseline > gpurun_out/c2_clk_$rep.log 2>&1
  PM_BENCH_NO_CLOCKS=1 python bench.py --config c2 --no-cpu-baseline > gpurun_out/c2_noclk_$rep.log 2>&1
done
for f in gpurun_out/c2_*.log; do echo "$f $(tail -1 $f | python -c 'import json,sys; l=json.loads(sys.stdin.read()); print(round(l["value"],1), l["clocks"])')"; done
