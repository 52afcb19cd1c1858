# A/B: fp32-X stream kernel stage height (16-row stages, 2 per warp) vs 32-row stages vs 7 warps
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_glm.py -m gpu -q -x > gpurun_out/t_glm.log 2>&1; echo "glm tests rc=$?" > gpurun_out/ab_f32tr.txt
tail -3 gpurun_out/t_glm.log >> gpurun_out/ab_f32tr.txt
for v in "tr16" "tr32 PM_STREAM_TR=32" "ncw7 PM_STREAM_NCW=7"; do
  set -- $v
  env $2 timeout 300 python bench.py --config c1f32 --steps 300 --no-cpu-baseline > gpurun_out/ab_f32tr_$1.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/ab_f32tr_$1.log').read().strip().splitlines()[-1]); print('$1', round(d['value'],1), round(d['roofline']['kernel_ms']*1000,1), 'us', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['roofline']['kernel'])" >> gpurun_out/ab_f32tr.txt 2>&1
done
cat gpurun_out/ab_f32tr.txt
