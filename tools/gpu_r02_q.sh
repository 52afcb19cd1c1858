# r02 pass Q: coalesced CTA-partial folds in the chain / diff kernels: tests + c2 line
O=gpurun_out/r02q
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_diff.py tests/test_gpu_protocols.py -m gpu -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$? $(tail -1 $O/pytest.log)" > $O/summary.txt
timeout 600 python bench.py --config c2 --no-cpu-baseline > $O/bench_c2.log 2>&1
timeout 600 python bench.py --config c2 --no-cpu-baseline > $O/bench_c2_again.log 2>&1
timeout 300 python tools/diff_latency.py > $O/diff_latency.log 2>&1
cat $O/summary.txt; tail -1 $O/diff_latency.log
