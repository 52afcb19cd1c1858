# final ncu --set full captures of the kernels as shipped: HB rows (8 self-producing warps, fused fold), c0 stream kernel
O=gpurun_out/r02al
mkdir -p $O
timeout 300 python tools/prof_hb.py > $O/plain_hb.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:hb_rows -s 2 -c 1 \
    -o $O/ncu_hb_final -f python tools/prof_hb.py > $O/ncu_hb.log 2>&1
timeout 300 python tools/prof_glm.py --n 100000 --k 32 > $O/plain_c0.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:glm_stream -s 3 -c 1 \
    -o $O/ncu_c0_final -f python tools/prof_glm.py --n 100000 --k 32 > $O/ncu_c0.log 2>&1
for r in $O/ncu_*.ncu-rep; do
  b=${r%.ncu-rep}
  ncu -i $r --page raw --csv > $b.raw.csv 2>/dev/null
  ncu -i $r --page details --csv > $b.details.csv 2>/dev/null
  rm -f $r
done
ls -la $O
