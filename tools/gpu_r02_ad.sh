O=gpurun_out/r02ad
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_protocols.py tests/test_gpu_hb.py -m gpu -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$? $(tail -1 $O/pytest.log)"
grep -E "^(FAILED|ERROR|E  )" $O/pytest.log | head -10
