mkdir -p gpurun_out
for n in 7 15; do
  PM_STREAM_NCW=$n timeout 300 python bench.py --config c1f32 --steps 300 --no-cpu-baseline > gpurun_out/ab_f32_ncw$n.log 2>&1
done
for f in gpurun_out/ab_f32_*.log; do
  python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value'],1), round(d['ms_per_step']*1000,1), 'us', round(d['roofline']['frac'],3))"
done > gpurun_out/ab_f32.txt
