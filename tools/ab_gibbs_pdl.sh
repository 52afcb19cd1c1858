# A/B: programmatic dependent launch of the packed Gibbs half-sweeps (PM_PDL=0 disables)
mkdir -p gpurun_out
: > gpurun_out/ab_gibbs_pdl.txt
for t in test_gpu_ising test_gpu_denoise test_gpu_dist; do
  timeout 900 python -m pytest tests/$t.py -m gpu -q -x > gpurun_out/tg_$t.log 2>&1; echo "$t rc=$? $(tail -1 gpurun_out/tg_$t.log)" >> gpurun_out/ab_gibbs_pdl.txt
done
for c in c4 c4potts; do
  for p in 1 0; do
    PM_PDL=$p timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/ab_gp_${c}_$p.log 2>&1
    python -c "import json; d=json.loads(open('gpurun_out/ab_gp_${c}_$p.log').read().strip().splitlines()[-1]); print('$c pdl=$p', round(d['value'],1), d['unit'], round(d['ms_per_step']*1000,2), 'us/step', 'e2e', round(d['e2e']['value'],1))" >> gpurun_out/ab_gibbs_pdl.txt 2>&1
  done
done
cat gpurun_out/ab_gibbs_pdl.txt
