# A/B: Potts code_bytes x + (x>>4) as one LEA.HI vs SHF+LOP3 (both ALU)
mkdir -p gpurun_out
: > gpurun_out/ab_potts_lea.txt
L=$PWD/paper_1310_1537_b200
timeout 900 python -m pytest tests/test_gpu_ising.py tests/test_gpu_dist.py -m gpu -q -x > gpurun_out/tg_ising.log 2>&1; echo "ising/dist tests rc=$? $(tail -1 gpurun_out/tg_ising.log)" >> gpurun_out/ab_potts_lea.txt
for rep in 1 2; do
for v in prev:$L/libpm_potts_prev.so lea:$L/libpmb200.so; do
  n=${v%%:*}; lib=${v#*:}
  PM_LIB_PATH=$lib timeout 600 python bench.py --config c4potts --no-cpu-baseline > gpurun_out/ab_lea_$n.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/ab_lea_$n.log').read().strip().splitlines()[-1]); print('c4potts rep$rep $n', round(d['value'],1), d['unit'], round(d['ms_per_step']*1000,2), 'us/step')" >> gpurun_out/ab_potts_lea.txt 2>&1
done
done
cat gpurun_out/ab_potts_lea.txt
