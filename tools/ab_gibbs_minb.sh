# A/B: register budget of the packed Gibbs kernel (min resident CTAs per SM 4 / 3 / 2 at NG >= 2)
mkdir -p gpurun_out
: > gpurun_out/ab_gibbs_minb.txt
L=$PWD/paper_1310_1537_b200
for c in c4 c4potts; do
  for v in 4:$L/libpmb200.so 3:$L/libpm_mb3.so 2:$L/libpm_mb2.so; do
    mb=${v%%:*}; lib=${v#*:}
    for ng in 4 2; do
      PM_GIBBS_NG=$ng PM_LIB_PATH=$lib timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/ab_mb_${c}_${mb}_$ng.log 2>&1
      python -c "import json; d=json.loads(open('gpurun_out/ab_mb_${c}_${mb}_$ng.log').read().strip().splitlines()[-1]); print('$c minb=$mb ng=$ng', round(d['value'],1), d['unit'], round(d['ms_per_step']*1000,2), 'us/step', 'sm_mhz', d['clocks']['sm_mhz'])" >> gpurun_out/ab_gibbs_minb.txt 2>&1
    done
  done
done
cat gpurun_out/ab_gibbs_minb.txt
