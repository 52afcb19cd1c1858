# A/B of the mbarrier try_wait suspend-time hint (default 1 ms, 0 = poll, 200 ns) on the
# streaming configs
mkdir -p gpurun_out
: > gpurun_out/ab_hint2.txt
L=$PWD/paper_1310_1537_b200
for c in c1f32 c1 c3 c0; do
  for lib in libpmb200.so libpm_h0.so libpm_h200.so; do
    PM_LIB_PATH=$L/$lib timeout 600 python bench.py --config $c --steps 300 --no-cpu-baseline > gpurun_out/bh_${c}_$lib.log 2>&1
    python -c "import json; d=json.loads(open('gpurun_out/bh_${c}_$lib.log').read().strip().splitlines()[-1]); print('$c $lib', round(d['value'],1), d['unit'], round(d['ms_per_step']*1000,2), 'us/step', round(d['roofline']['frac'],3))" >> gpurun_out/ab_hint2.txt 2>&1
  done
done
cat gpurun_out/ab_hint2.txt
