# A/B: Potts packed path, carry-count thresholds + raw prmt (vs lane table alone: 107.5 us ng4 / 105.3 us ng2)
mkdir -p gpurun_out
: > gpurun_out/ab_potts_carry.txt
for t in test_gpu_ising test_gpu_denoise test_gpu_dist; do
  timeout 900 python -m pytest tests/$t.py -m gpu -q -x > gpurun_out/tg_$t.log 2>&1; echo "$t rc=$? $(tail -1 gpurun_out/tg_$t.log)" >> gpurun_out/ab_potts_carry.txt
done
run() {  # name, env...
  n=$1; shift
  env "$@" timeout 600 python bench.py --config c4potts --no-cpu-baseline > gpurun_out/ab_pc_$n.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/ab_pc_$n.log').read().strip().splitlines()[-1]); print('$n', round(d['value'],1), d['unit'], round(d['ms_per_step']*1000,2), 'us/step', 'e2e', round(d['e2e']['value'],1))" >> gpurun_out/ab_potts_carry.txt 2>&1
}
run carry_ng4 PM_GIBBS_NG=4
run carry_ng2 PM_GIBBS_NG=2
run carry_ng1 PM_GIBBS_NG=1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gibbs_packed -s 2 -c 1 -o gpurun_out/ncu_potts_carry -f env PM_GIBBS_NG=2 python tools/prof_ising.py --potts > gpurun_out/ncu_pc.log 2>&1
cat gpurun_out/ab_potts_carry.txt
