# r02 pass D: after the coalesced fold / compile-time MULTI / barrier placement
O=gpurun_out/r02d
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_glm.py tests/test_gpu_protocols.py tests/test_gpu_hb.py tests/test_gpu_dist.py tests/test_gpu_diff.py -m gpu -x -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$? $(tail -1 $O/pytest.log)" > $O/summary.txt
for v in default NO_FINALIZE PHASES; do
  if [ $v = default ]; then L=""; else L="PM_LIB_PATH=$PWD/paper_1310_1537_b200/libpmb200_$v.so"; fi
  env $L timeout 300 python tools/c0_breakdown.py --tag $v >> $O/c0_breakdown.jsonl 2>> $O/c0_breakdown.err
done
for t in 1 2 4; do timeout 300 python tools/c0_breakdown.py --tag tps$t --tune stream_tps=$t >> $O/c0_breakdown.jsonl 2>> $O/c0_tps.err; done
timeout 300 python tools/c0_breakdown.py --tag rows --tune glm_rows=1 >> $O/c0_breakdown.jsonl 2>> $O/c0_tps.err
for t in 2 4 8; do timeout 300 python tools/c0_breakdown.py --tag rows_tps$t --tune glm_rows=1 --tune rows_tps=$t >> $O/c0_breakdown.jsonl 2>> $O/c0_tps.err; done
timeout 600 python bench.py --config c0 --no-cpu-baseline > $O/bench_c0.log 2>&1; echo "c0 rc=$?" >> $O/summary.txt
timeout 600 python bench.py --config c1 --no-cpu-baseline --steps 300 > $O/bench_c1.log 2>&1; echo "c1 rc=$?" >> $O/summary.txt
timeout 600 python bench.py --config c1f32 --no-cpu-baseline --steps 300 > $O/bench_c1f32.log 2>&1; echo "c1f32 rc=$?" >> $O/summary.txt
timeout 600 python bench.py --config c4potts --steps 1000 --warmup 10 --no-cpu-baseline --tune gibbs_smem=1 > $O/c4p_smem1.log 2>&1
cat $O/summary.txt
