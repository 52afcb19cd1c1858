O=gpurun_out/r02ak
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_diff.py tests/test_gpu_protocols.py tests/test_gpu_reference_suite.py -m gpu -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$? $(tail -1 $O/pytest.log)"
timeout 300 python tools/diff_latency.py 2>&1 | tail -1
