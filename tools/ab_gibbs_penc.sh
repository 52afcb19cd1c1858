# A/B: packed Potts bytes stored as the compact code (no per-neighbour lookups) vs states
mkdir -p gpurun_out
: > gpurun_out/ab_gibbs_penc.txt
L=$PWD/paper_1310_1537_b200
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/tg_ks.log 2>&1; echo "ising/dist/denoise tests rc=$? $(tail -1 gpurun_out/tg_ks.log)" >> gpurun_out/ab_gibbs_penc.txt
for rep in 1 2; do
for c in c4 c4potts; do
for v in before:$L/libpm_before_enc.so enc:$L/libpmb200.so; do
  n=${v%%:*}; lib=${v#*:}
  PM_LIB_PATH=$lib timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/ab_penc_$n.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/ab_penc_$n.log').read().strip().splitlines()[-1]); print('$c rep$rep $n', round(d['value'],1), d['unit'], round(d['ms_per_step']*1000,2), 'us/step')" >> gpurun_out/ab_gibbs_penc.txt 2>&1
done
done
done
cat gpurun_out/ab_gibbs_penc.txt
