# A/B: Ising packed kernel at NG=2 with 4 / 5 / 6 resident CTAs per SM; new defaults (Ising NG=2, Potts NG=4 + 3 CTAs/SM)
mkdir -p gpurun_out
: > gpurun_out/ab_gibbs_minb2.txt
L=$PWD/paper_1310_1537_b200
timeout 900 python -m pytest tests/test_gpu_ising.py tests/test_gpu_dist.py tests/test_gpu_denoise.py -m gpu -q -x > gpurun_out/tg_ising.log 2>&1; echo "ising/dist/denoise tests rc=$? $(tail -1 gpurun_out/tg_ising.log)" >> gpurun_out/ab_gibbs_minb2.txt
for rep in 1 2; do
for v in 4:$L/libpmb200.so 5:$L/libpm_mi5.so 6:$L/libpm_mi6.so; do
  mb=${v%%:*}; lib=${v#*:}
  PM_LIB_PATH=$lib timeout 600 python bench.py --config c4 --no-cpu-baseline > gpurun_out/ab_mi_${mb}.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/ab_mi_${mb}.log').read().strip().splitlines()[-1]); print('c4 rep$rep minb=$mb ng=2', round(d['value'],1), d['unit'], round(d['ms_per_step']*1000,2), 'us/step', 'sm_mhz', d['clocks']['sm_mhz'])" >> gpurun_out/ab_gibbs_minb2.txt 2>&1
done
done
timeout 600 python bench.py --config c4potts --no-cpu-baseline > gpurun_out/ab_mi_potts.log 2>&1
python -c "import json; d=json.loads(open('gpurun_out/ab_mi_potts.log').read().strip().splitlines()[-1]); print('c4potts default', round(d['value'],1), d['unit'], round(d['ms_per_step']*1000,2), 'us/step')" >> gpurun_out/ab_gibbs_minb2.txt 2>&1
cat gpurun_out/ab_gibbs_minb2.txt
