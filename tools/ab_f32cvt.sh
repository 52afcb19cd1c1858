# A/B: fp32-X widening by integer ops (default build) vs F2F.F64.F32 (libpm_f2f.so, -DPM_F32_F2F)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_glm.py -m gpu -q -x > gpurun_out/t_glm.log 2>&1; echo "glm tests rc=$?" > gpurun_out/ab_f32cvt.txt
for lib in default f2f; do
  for n in 7 15; do
    if [ $lib = f2f ]; then export PM_LIB_PATH=$PWD/paper_1310_1537_b200/libpm_f2f.so; else unset PM_LIB_PATH; fi
    PM_STREAM_NCW=$n timeout 300 python bench.py --config c1f32 --steps 300 --no-cpu-baseline > gpurun_out/ab_f32cvt_${lib}_$n.log 2>&1
  done
done
unset PM_LIB_PATH
for f in gpurun_out/ab_f32cvt_*.log; do
  python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value'],1), round(d['roofline']['kernel_ms']*1000,1), 'us', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" >> gpurun_out/ab_f32cvt.txt 2>&1
done
timeout 300 python tools/prof_glm.py --f32 > gpurun_out/prof_f32.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:glm_stream -s 2 -c 1 \
    -o gpurun_out/glm_stream_f32_full -f python tools/prof_glm.py --f32 > gpurun_out/ncu_f32.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ab_f32cvt.txt
cat gpurun_out/ab_f32cvt.txt
