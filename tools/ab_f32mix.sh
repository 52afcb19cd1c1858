# A/B of the fp32 widening in the pairs layout: integer (default) / mixed F2F+integer / all F2F
mkdir -p gpurun_out
L=$PWD/paper_1310_1537_b200
PM_LIB_PATH=$L/libpm_mix.so timeout 900 python -m pytest tests/test_gpu_glm.py -m gpu -q -x -k fp32 > gpurun_out/t_glm_mix.log 2>&1; echo "mix fp32 tests rc=$?" > gpurun_out/ab_f32mix.txt
for v in "int15 libpmb200.so" "mix15 libpm_mix.so" "f2f15 libpm_f2f.so" "int7 libpmb200.so PM_STREAM_NCW=7" "mix7 libpm_mix.so PM_STREAM_NCW=7"; do
  set -- $v
  env PM_LIB_PATH=$L/$2 $3 timeout 300 python bench.py --config c1f32 --steps 300 --no-cpu-baseline > gpurun_out/ab_f32m_$1.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/ab_f32m_$1.log').read().strip().splitlines()[-1]); print('$1', round(d['value'],1), round(d['roofline']['kernel_ms']*1000,1), 'us', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" >> gpurun_out/ab_f32mix.txt 2>&1
done
cat gpurun_out/ab_f32mix.txt
