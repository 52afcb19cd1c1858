O=gpurun_out/r02ai
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_hb.py tests/test_gpu_hb_sweep.py tests/test_gpu_protocols.py tests/test_gpu_reference_suite.py -m gpu -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$? $(tail -1 $O/pytest.log)"
timeout 600 python bench.py --config c3 > $O/bench_c3.log 2>&1
tail -1 $O/bench_c3.log | python -c "
import sys,json
l=json.loads(sys.stdin.read()); r=l['roofline']; print('c3', round(l['value'],1), round(l['ms_per_step']*1e3,2), 'us frac', round(r['frac'],3), 'e2e', round(l['e2e']['value'],1), r.get('kernel'))"
