# A/B: producer lanes issuing the TMA bulk copies of the GLM stream kernel (1 / 2 / 4)
mkdir -p gpurun_out
: > gpurun_out/ab_nprod.txt
L=$PWD/paper_1310_1537_b200
for lib in libpm_np2.so libpm_np4.so; do
  PM_LIB_PATH=$L/$lib timeout 900 python -m pytest tests/test_gpu_glm.py -m gpu -q -x > gpurun_out/tn_$lib.log 2>&1; echo "glm tests $lib rc=$? $(tail -1 gpurun_out/tn_$lib.log)" >> gpurun_out/ab_nprod.txt
done
for c in c1f32 c1 c0; do
  for lib in libpmb200.so libpm_np2.so libpm_np4.so; do
    PM_LIB_PATH=$L/$lib timeout 600 python bench.py --config $c --steps 300 --no-cpu-baseline > gpurun_out/bn_${c}_$lib.log 2>&1
    python -c "import json; d=json.loads(open('gpurun_out/bn_${c}_$lib.log').read().strip().splitlines()[-1]); print('$c $lib', round(d['value'],1), d['unit'], round(d['ms_per_step']*1000,2), 'us/step', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" >> gpurun_out/ab_nprod.txt 2>&1
  done
done
cat gpurun_out/ab_nprod.txt
