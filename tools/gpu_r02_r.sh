# r02 pass R: chain kernel own grid barrier A/B + chain tests
O=gpurun_out/r02r
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_diff.py -m gpu -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$? $(tail -1 $O/pytest.log)" > $O/summary.txt
for t in 1 0 1 0; do timeout 600 python bench.py --config c2 --no-cpu-baseline --tune chain_own_barrier=$t >> $O/c2_bar$t.log 2>&1; done
cat $O/summary.txt
