O=gpurun_out/r02af
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_glm.py tests/test_gpu_protocols.py -m gpu -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$? $(tail -1 $O/pytest.log)"
timeout 600 python bench.py --config c1f32 --no-cpu-baseline --steps 20 --warmup 3 > $O/c1f32.log 2>&1
tail -1 $O/c1f32.log | python -c "
import sys,json
l=json.loads(sys.stdin.read()); r=l['roofline']; print('c1f32', round(l['value'],1), round(l['ms_per_step'],4), 'frac', round(r['frac'],3), l['clocks'])"
