# r02 pass C: stream-kernel changes (tiles per stage, prologue overlap, single-pass fold):
# GLM/HB/dist parity tests, c0 breakdown over the A/B builds, c0 / c1 / c1f32 lines
O=gpurun_out/r02c
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_glm.py tests/test_gpu_hb.py tests/test_gpu_dist.py tests/test_gpu_diff.py -m gpu -x -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$? $(tail -1 $O/pytest.log)" > $O/summary.txt
for v in default EMPTY NO_FINALIZE PHASES OUT_DEVICE; do
  if [ $v = default ]; then L=""; else L="PM_LIB_PATH=$PWD/paper_1310_1537_b200/libpmb200_$v.so"; fi
  env $L timeout 300 python tools/c0_breakdown.py --tag $v >> $O/c0_breakdown.jsonl 2>> $O/c0_breakdown.err
done
for t in 1 2 3 4; do timeout 300 python tools/c0_breakdown.py --tag tps$t --tune stream_tps=$t >> $O/c0_breakdown.jsonl 2>> $O/c0_tps.err; done
timeout 600 python bench.py --config c0 --no-cpu-baseline > $O/bench_c0.log 2>&1; echo "c0 rc=$?" >> $O/summary.txt
timeout 600 python bench.py --config c1 --no-cpu-baseline --steps 300 > $O/bench_c1.log 2>&1; echo "c1 rc=$?" >> $O/summary.txt
timeout 600 python bench.py --config c1f32 --no-cpu-baseline --steps 300 > $O/bench_c1f32.log 2>&1; echo "c1f32 rc=$?" >> $O/summary.txt
cat $O/summary.txt
