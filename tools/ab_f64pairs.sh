# A/B: fp64 stream kernel consumer layout, column pairs + XOR rows (default) vs column per lane
mkdir -p gpurun_out
: > gpurun_out/ab_f64pairs.txt
timeout 900 python -m pytest tests/test_gpu_glm.py tests/test_gpu_dist.py -m gpu -q -x > gpurun_out/t_glm.log 2>&1; echo "glm+dist tests rc=$? $(tail -1 gpurun_out/t_glm.log)" >> gpurun_out/ab_f64pairs.txt
for c in c1 c0 c1f32; do
  for p in 1 0; do
    PM_F64_PAIRS=$p timeout 600 python bench.py --config $c --steps 300 --no-cpu-baseline > gpurun_out/bp_${c}_$p.log 2>&1
    python -c "import json; d=json.loads(open('gpurun_out/bp_${c}_$p.log').read().strip().splitlines()[-1]); print('$c pairs=$p', round(d['value'],1), d['unit'], round(d['roofline']['kernel_ms']*1000,1), 'us kernel', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])" >> gpurun_out/ab_f64pairs.txt 2>&1
  done
done
timeout 300 python tools/prof_glm.py > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:glm_stream -s 2 -c 1 \
    -o gpurun_out/glm_stream_f64pairs -f python tools/prof_glm.py > gpurun_out/ncu_f64p.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ab_f64pairs.txt
cat gpurun_out/ab_f64pairs.txt
