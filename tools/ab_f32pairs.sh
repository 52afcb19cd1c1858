# A/B: fp32-X pairs consumer layout vs column-per-lane, 15 vs 7 consumer warps; glm tests first
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_glm.py -m gpu -q -x > gpurun_out/t_glm.log 2>&1; echo "glm tests rc=$?" > gpurun_out/ab_f32pairs.txt
tail -3 gpurun_out/t_glm.log >> gpurun_out/ab_f32pairs.txt
for v in "pairs15 PM_F32_PAIRS=1" "cols15 PM_F32_PAIRS=0" "pairs7 PM_STREAM_NCW=7" "cols7 PM_F32_PAIRS=0,PM_STREAM_NCW=7"; do
  set -- $v
  env $(echo $2 | tr ',' ' ') timeout 300 python bench.py --config c1f32 --steps 300 --no-cpu-baseline > gpurun_out/ab_f32p_$1.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/ab_f32p_$1.log').read().strip().splitlines()[-1]); print('$1', round(d['value'],1), round(d['roofline']['kernel_ms']*1000,1), 'us', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['roofline']['kernel'])" >> gpurun_out/ab_f32pairs.txt 2>&1
done
timeout 300 python tools/prof_glm.py --f32 > gpurun_out/prof_f32.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:glm_stream -s 2 -c 1 \
    -o gpurun_out/glm_stream_f32p_full -f python tools/prof_glm.py --f32 > gpurun_out/ncu_f32.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ab_f32pairs.txt
cat gpurun_out/ab_f32pairs.txt
