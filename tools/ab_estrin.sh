# A/B: Estrin vs Horner exp polynomial (pm_math.cuh) across the GLM configs; tests on Estrin
mkdir -p gpurun_out
: > gpurun_out/ab_estrin.txt
for t in test_gpu_glm test_gpu_diff test_gpu_hb test_gpu_hb_sweep; do
  timeout 900 python -m pytest tests/$t.py -m gpu -q -x > gpurun_out/te_$t.log 2>&1; echo "$t rc=$? $(tail -1 gpurun_out/te_$t.log)" >> gpurun_out/ab_estrin.txt
done
L=$PWD/paper_1310_1537_b200
for c in c1f32 c3 c2 c0 c1; do
  for lib in libpmb200.so libpm_horner.so; do
    PM_LIB_PATH=$L/$lib timeout 600 python bench.py --config $c --steps 200 --no-cpu-baseline > gpurun_out/be_${c}_$lib.log 2>&1
    python -c "import json; d=json.loads(open('gpurun_out/be_${c}_$lib.log').read().strip().splitlines()[-1]); print('$c $lib', round(d['value'],1), d['unit'], round(d['ms_per_step']*1000,2), 'us/step', round(d['roofline']['frac'],3))" >> gpurun_out/ab_estrin.txt 2>&1
  done
done
cat gpurun_out/ab_estrin.txt
