O=gpurun_out/r02ab
mkdir -p $O
for i in 1 2 3; do for t in "hb_mapped_out=0" "hb_mapped_out=1"; do
  echo "== $t" >> $O/c3.log
  timeout 600 python bench.py --config c3 --no-cpu-baseline --tune $t >> $O/c3.log 2>&1
done; done
python - <<'PY'
import json
tag=None
for line in open('gpurun_out/r02ab/c3.log'):
    if line.startswith('=='): tag=line.strip()
    elif line.startswith('{'):
        l=json.loads(line); print(tag, 'device us', round(l['ms_per_step']*1e3,2), 'e2e', round(l['e2e']['value'],1), round(1e6/l['e2e']['value'],1), 'us')
PY
