mkdir -p gpurun_out
: > gpurun_out/ab_hbpair.txt
timeout 900 python -m pytest tests/test_gpu_hb.py -m gpu -q -x > gpurun_out/thp.log 2>&1; echo "hb tests rc=$? $(tail -1 gpurun_out/thp.log)" >> gpurun_out/ab_hbpair.txt
L=$PWD/paper_1310_1537_b200
for v in "pair libpmb200.so" "single libpm_hp0.so" "pair2 libpmb200.so" "single2 libpm_hp0.so"; do
  set -- $v
  PM_LIB_PATH=$L/$2 timeout 300 python bench.py --config c3 --steps 500 --no-cpu-baseline > gpurun_out/bhp_$1.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/bhp_$1.log').read().strip().splitlines()[-1]); print('$1', round(d['value'],1), round(d['ms_per_step']*1000,2), 'us', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" >> gpurun_out/ab_hbpair.txt 2>&1
done
cat gpurun_out/ab_hbpair.txt
