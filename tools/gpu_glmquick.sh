mkdir -p gpurun_out
: > gpurun_out/glmq.txt
timeout 900 python -m pytest tests/test_gpu_glm.py tests/test_gpu_dist.py tests/test_gpu_diff.py -m gpu -q -x > gpurun_out/tq.log 2>&1; echo "tests rc=$? $(tail -1 gpurun_out/tq.log)" >> gpurun_out/glmq.txt
for c in c1f32 c1; do
  timeout 600 python bench.py --config $c --steps 300 --no-cpu-baseline > gpurun_out/bq_$c.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/bq_$c.log').read().strip().splitlines()[-1]); print('$c', round(d['value'],1), round(d['roofline']['kernel_ms']*1000,1), 'us', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['roofline']['kernel'])" >> gpurun_out/glmq.txt 2>&1
done
cat gpurun_out/glmq.txt
