# A/B of the row-per-lane HB kernel knobs (consumer warps, tiles per stage)
mkdir -p gpurun_out
for cfg in "7 1" "7 2" "7 4" "15 1" "15 2" "15 4"; do
  set -- $cfg
  PM_HB_ROWS_NCW=$1 PM_HB_ROWS_TPS=$2 timeout 300 python bench.py --config c3 --steps 300 --no-cpu-baseline \
    > gpurun_out/hbrows_ncw$1_tps$2.log 2>&1
done
for f in gpurun_out/hbrows_*.log; do
  python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value'],1), round(d['ms_per_step']*1000,1), 'us', round(d['roofline']['frac'],3))"
done > gpurun_out/ab_hb_rows.txt
