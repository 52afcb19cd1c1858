# groups-per-thread re-check after the packed encodings (env override of the defaults)
: > gpurun_out/ab_ng_final.txt
for c in c4 c4potts; do for ng in 1 2 4; do
  PM_GIBBS_NG=$ng timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/ab_ngf.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/ab_ngf.log').read().strip().splitlines()[-1]); print('$c ng=$ng', round(d['value'],1), d['unit'], round(d['ms_per_step']*1000,2), 'us/step')" >> gpurun_out/ab_ng_final.txt 2>&1
done; done
cat gpurun_out/ab_ng_final.txt
