# last check on the clean build: smoke, every GPU test, default bench line
O=gpurun_out/r02last
mkdir -p $O
timeout 600 python __graft_entry__.py --smoke > $O/smoke.log 2>&1; echo "smoke rc=$? $(tail -1 $O/smoke.log)" > $O/summary.txt
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$? $(tail -1 $O/pytest.log)" >> $O/summary.txt
timeout 900 python bench.py --steps 20 --warmup 3 > $O/bench_default.log 2>&1; echo "bench rc=$?" >> $O/summary.txt
timeout 900 python bench.py --impl reference --steps 20 --warmup 3 > $O/bench_reference.log 2>&1; echo "reference rc=$?" >> $O/summary.txt
cat $O/summary.txt; tail -c 400 $O/bench_default.log
