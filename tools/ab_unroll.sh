# A/B: pairs consumer sub-tile interleaving (unroll 2) and rows per sub-tile for 7 consumer warps
mkdir -p gpurun_out
: > gpurun_out/ab_unroll.txt
L=$PWD/paper_1310_1537_b200
for v in "base15 libpmb200.so" "base7 libpmb200.so PM_STREAM_NCW=7" "u2r8_7 libpm_u2.so PM_STREAM_NCW=7" "u2r16_7 libpm_u2r16.so PM_STREAM_NCW=7"; do
  set -- $v
  env PM_LIB_PATH=$L/$2 $3 timeout 600 python bench.py --config c1f32 --steps 300 --no-cpu-baseline > gpurun_out/bu_$1.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/bu_$1.log').read().strip().splitlines()[-1]); print('c1f32 $1', round(d['value'],1), round(d['roofline']['kernel_ms']*1000,1), 'us', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" >> gpurun_out/ab_unroll.txt 2>&1
done
for v in "base libpmb200.so" "u2r16 libpm_u2r16.so"; do
  set -- $v
  env PM_LIB_PATH=$L/$2 timeout 600 python bench.py --config c1 --steps 300 --no-cpu-baseline > gpurun_out/bu1_$1.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/bu1_$1.log').read().strip().splitlines()[-1]); print('c1 $1', round(d['value'],1), round(d['roofline']['kernel_ms']*1000,1), 'us', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" >> gpurun_out/ab_unroll.txt 2>&1
done
PM_LIB_PATH=$L/libpm_u2r16.so timeout 900 python -m pytest tests/test_gpu_glm.py -m gpu -q -x > gpurun_out/tu.log 2>&1; echo "glm tests u2r16 rc=$? $(tail -1 gpurun_out/tu.log)" >> gpurun_out/ab_unroll.txt
cat gpurun_out/ab_unroll.txt
