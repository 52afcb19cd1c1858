# r02: GPU tests + c0 fixed-cost breakdown after the finalize changes + c0/c2/c3 bench lines
O=gpurun_out/r02c
mkdir -p $O
for v in default EMPTY NO_FINALIZE; do
  if [ $v = default ]; then L=""; else L="PM_LIB_PATH=$PWD/paper_1310_1537_b200/libpmb200_$v.so"; fi
  env $L timeout 300 python tools/c0_breakdown.py --tag $v >> $O/c0_breakdown.jsonl 2>> $O/c0_breakdown.err
done
timeout 600 python bench.py --config c0 --steps 200 --warmup 10 > $O/bench_c0.log 2>&1
timeout 600 python bench.py --config c2 --steps 20 --warmup 3 > $O/bench_c2.log 2>&1
timeout 600 python bench.py --config c3 --steps 200 --warmup 5 > $O/bench_c3.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=20 > $O/pytest.log 2>&1
tail -3 $O/pytest.log
