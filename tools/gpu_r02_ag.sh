O=gpurun_out/r02ag
mkdir -p $O
for t in "hb_fused=0" "hb_fused=1" "hb_rows_stages=8" "hb_rows_stages=16" "hb_rows_stages=24" "hb_contig=0" "pdl=0"; do
  echo "== $t" >> $O/c3.log
  timeout 600 python bench.py --config c3 --no-cpu-baseline --tune $t >> $O/c3.log 2>&1
done
python - <<'PY'
import json
tag=None
for line in open('gpurun_out/r02ag/c3.log'):
    if line.startswith('=='): tag=line.strip()
    elif line.startswith('{'):
        l=json.loads(line); print(tag, 'device us', round(l['ms_per_step']*1e3,2), 'frac', round(l['roofline']['frac'],3), 'e2e us', round(1e6/l['e2e']['value'],1), l['roofline'].get('kernel','')[:70])
PY
