# r02 pass W: Python hot-path trims: breakdown + GLM tests + reference suite + c0 line
O=gpurun_out/r02w
mkdir -p $O
timeout 300 python tools/e2e_breakdown.py > $O/e2e_c0.json 2> $O/e2e.err
timeout 1500 python -m pytest tests/test_gpu_glm.py tests/test_abi.py tests/test_gpu_dist.py tests/test_gpu_reference_suite.py tests/test_gpu_diff.py -m gpu -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$? $(tail -1 $O/pytest.log)" > $O/summary.txt
timeout 600 python bench.py --config c0 --no-cpu-baseline > $O/bench_c0.log 2>&1
cat $O/e2e_c0.json $O/summary.txt
