# r02 pass E: fold with fixed 4 chunks (finer phase stamps, with and without mapped-host output),
# config-4 end-to-end breakdown, GLM + protocol tests
O=gpurun_out/r02e
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_glm.py tests/test_gpu_protocols.py tests/test_gpu_dist.py -m gpu -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$? $(tail -1 $O/pytest.log)" > $O/summary.txt
for v in default PHASES PHOD; do
  if [ $v = default ]; then L=""; else L="PM_LIB_PATH=$PWD/paper_1310_1537_b200/libpmb200_$v.so"; fi
  env $L timeout 300 python tools/c0_breakdown.py --tag $v >> $O/c0_breakdown.jsonl 2>> $O/c0_breakdown.err
done
timeout 900 python tools/c4_e2e_breakdown.py > $O/c4_e2e.jsonl 2> $O/c4_e2e.err
timeout 600 python bench.py --config c0 --no-cpu-baseline > $O/bench_c0.log 2>&1; echo "c0 rc=$?" >> $O/summary.txt
cat $O/summary.txt
