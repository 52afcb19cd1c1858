# r02 pass M: row-dot default; F2F share A/B (0 / 1 / 2 leading pairs per gradient row); GLM + protocol tests
O=gpurun_out/r02m
mkdir -p $O
timeout 600 python bench.py --config c1f32 --no-cpu-baseline --steps 300 > $O/c1f32_f2f1.log 2>&1
for v in 0 2; do
  PM_LIB_PATH=$PWD/paper_1310_1537_b200/libpmb200_F2F$v.so timeout 600 python bench.py --config c1f32 --no-cpu-baseline --steps 300 > $O/c1f32_f2f$v.log 2>&1
done
timeout 600 python bench.py --config c1f32 --no-cpu-baseline --steps 300 > $O/c1f32_f2f1_again.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_glm.py tests/test_gpu_protocols.py tests/test_gpu_dist.py tests/test_gpu_multiproc.py -m gpu -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$? $(tail -1 $O/pytest.log)" > $O/summary.txt
cat $O/summary.txt
