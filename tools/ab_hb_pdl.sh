# A/B: programmatic dependent launch for the HB rows kernel (PM_PDL=0 disables)
mkdir -p gpurun_out
: > gpurun_out/ab_hb_pdl.txt
timeout 900 python -m pytest tests/test_gpu_hb.py -m gpu -q -x > gpurun_out/t_hb.log 2>&1; echo "hb tests rc=$? $(tail -1 gpurun_out/t_hb.log)" >> gpurun_out/ab_hb_pdl.txt
PM_HB_FUSED=0 timeout 900 python -m pytest tests/test_gpu_hb.py -m gpu -q -x > gpurun_out/t_hb0.log 2>&1; echo "hb tests unfused rc=$? $(tail -1 gpurun_out/t_hb0.log)" >> gpurun_out/ab_hb_pdl.txt
for v in "pdl_fused PM_PDL=1" "pdl_unfused PM_HB_FUSED=0" "nopdl_unfused PM_PDL=0,PM_HB_FUSED=0" "pdl_unfused2 PM_HB_FUSED=0"; do
  set -- $v
  env $(echo $2 | tr "," " ") timeout 300 python bench.py --config c3 --steps 500 --no-cpu-baseline > gpurun_out/ab_hbp_$1.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/ab_hbp_$1.log').read().strip().splitlines()[-1]); print('$1', round(d['value'],1), round(d['ms_per_step']*1000,2), 'us', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value'],1))" >> gpurun_out/ab_hb_pdl.txt 2>&1
done
cat gpurun_out/ab_hb_pdl.txt
