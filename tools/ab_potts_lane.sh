# A/B: Potts packed path, lane-replicated compact threshold table (new) vs 625-entry uint4 table (old lib)
mkdir -p gpurun_out
: > gpurun_out/ab_potts_lane.txt
for t in test_gpu_ising test_gpu_denoise test_gpu_dist; do
  timeout 900 python -m pytest tests/$t.py -m gpu -q -x > gpurun_out/tg_$t.log 2>&1; echo "$t rc=$? $(tail -1 gpurun_out/tg_$t.log)" >> gpurun_out/ab_potts_lane.txt
done
run() {  # name, env...
  n=$1; shift
  env "$@" timeout 600 python bench.py --config c4potts --no-cpu-baseline > gpurun_out/ab_pl_$n.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/ab_pl_$n.log').read().strip().splitlines()[-1]); print('$n', round(d['value'],1), d['unit'], round(d['ms_per_step']*1000,2), 'us/step', 'e2e', round(d['e2e']['value'],1))" >> gpurun_out/ab_potts_lane.txt 2>&1
}
run old PM_LIB_PATH=$PWD/paper_1310_1537_b200/libpm_potts_old.so
run new_ng4 PM_GIBBS_NG=4
run new_ng2 PM_GIBBS_NG=2
run new_ng1 PM_GIBBS_NG=1
run old_ng2 PM_GIBBS_NG=2 PM_LIB_PATH=$PWD/paper_1310_1537_b200/libpm_potts_old.so
timeout 600 python bench.py --config c4 --no-cpu-baseline > gpurun_out/ab_pl_c4.log 2>&1; tail -1 gpurun_out/ab_pl_c4.log | cut -c1-250 >> gpurun_out/ab_potts_lane.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gibbs_packed -s 2 -c 1 -o gpurun_out/ncu_potts_new -f python tools/prof_ising.py --potts > gpurun_out/ncu_pn.log 2>&1
PM_LIB_PATH=$PWD/paper_1310_1537_b200/libpm_potts_old.so timeout 600 ncu --set full --clock-control none -k regex:gibbs_packed -s 2 -c 1 -o gpurun_out/ncu_potts_old -f python tools/prof_ising.py --potts > gpurun_out/ncu_po.log 2>&1
cat gpurun_out/ab_potts_lane.txt
