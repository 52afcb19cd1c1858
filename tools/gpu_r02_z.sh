# r02 pass Z: HB evaluation host path (fused staging + finiteness, raw-address call): tests + c3 line
O=gpurun_out/r02z
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_hb.py tests/test_gpu_hb_sweep.py tests/test_gpu_reference_suite.py -m gpu -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$? $(tail -1 $O/pytest.log)" > $O/summary.txt
for i in 1 2; do timeout 600 python bench.py --config c3 --no-cpu-baseline >> $O/bench_c3.log 2>&1; done
cat $O/summary.txt; grep '^{' $O/bench_c3.log | python -c "
import sys,json
for line in sys.stdin:
    l=json.loads(line); print('c3', round(l['value'],1), 'e2e', round(l['e2e']['value'],1), round(1e6/l['e2e']['value'],1), 'us')"
