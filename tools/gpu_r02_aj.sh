O=gpurun_out/r02aj
mkdir -p $O
for t in "chain_spec=4" "chain_blocks_per_sm=1" "chain_blocks_per_sm=3" "chain_blocks_per_sm=4" "chain_spec=2" "chain_spec=3" "chain_spec=5" "chain_spec=6" "chain_unroll=1" "chain_unroll=4"; do
  echo "== $t" >> $O/c2.log
  timeout 600 python bench.py --config c2 --no-cpu-baseline --steps 10 --tune $t >> $O/c2.log 2>&1
done
python - <<'PY'
import json
tag=None
for line in open('gpurun_out/r02aj/c2.log'):
    if line.startswith('=='): tag=line.strip()
    elif line.startswith('{'):
        l=json.loads(line); print(tag, round(l['value'],1), 'it/s', round(l['ms_per_step'],3), 'ms')
PY
