# r02 pass T: host-side rewrites (instrumentation, perf grid runner, slice sampler): every GPU test
O=gpurun_out/r02t
mkdir -p $O
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$? $(tail -1 $O/pytest.log)" > $O/summary.txt
timeout 600 python bench.py --config c0 --no-cpu-baseline > $O/bench_c0.log 2>&1
cat $O/summary.txt
