# A/B: HB fused fold (one launch) vs hb_fold_kernel; contiguous vs round-robin warp ranges
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_hb.py tests/test_gpu_hb_sweep.py -m gpu -q -x > gpurun_out/t_hb.log 2>&1; echo "hb tests rc=$?" > gpurun_out/ab_hb_fused.txt
tail -1 gpurun_out/t_hb.log >> gpurun_out/ab_hb_fused.txt
PM_HB_FUSED=0 timeout 900 python -m pytest tests/test_gpu_hb.py -m gpu -q -x > gpurun_out/t_hb0.log 2>&1; echo "hb tests unfused rc=$?" >> gpurun_out/ab_hb_fused.txt
for v in "fused PM_HB_FUSED=1" "unfused PM_HB_FUSED=0" "fused_rr PM_HB_CONTIG=0" "fused2 PM_HB_FUSED=1"; do
  set -- $v
  env $2 timeout 300 python bench.py --config c3 --steps 500 --no-cpu-baseline > gpurun_out/ab_hbf_$1.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/ab_hbf_$1.log').read().strip().splitlines()[-1]); print('$1', round(d['value'],1), round(d['ms_per_step']*1000,2), 'us', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value'],1))" >> gpurun_out/ab_hb_fused.txt 2>&1
done
cat gpurun_out/ab_hb_fused.txt
