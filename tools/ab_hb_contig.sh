# A/B: HB rows kernel unit assignment, round-robin (0) vs contiguous per warp (1); ncu of the default
mkdir -p gpurun_out
: > gpurun_out/ab_hb_contig.txt
for c in 0 1 0 1; do
  PM_HB_CONTIG=$c timeout 300 python bench.py --config c3 --steps 500 --no-cpu-baseline > gpurun_out/ab_hb_c$c.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/ab_hb_c$c.log').read().strip().splitlines()[-1]); print('contig=$c', round(d['value'],1), round(d['ms_per_step']*1000,2), 'us', round(d['roofline']['frac'],3))" >> gpurun_out/ab_hb_contig.txt 2>&1
done
timeout 300 python tools/prof_hb.py > gpurun_out/prof_hb.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hb_rows -s 2 -c 1 \
    -o gpurun_out/hb_rows_full -f python tools/prof_hb.py > gpurun_out/ncu_hb.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ab_hb_contig.txt
cat gpurun_out/ab_hb_contig.txt
