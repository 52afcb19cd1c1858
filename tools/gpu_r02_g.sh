# r02 pass G: ncu source-level capture of the fp32-X row-dot consumer (15 warps)
O=gpurun_out/r02g
mkdir -p $O
timeout 300 python tools/prof_glm.py --f32 --tune f32_pairs=3 --tune stream_ncw=15 > $O/plain.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:glm_stream -s 3 -c 1 \
    -o $O/ncu_rowdot15 -f python tools/prof_glm.py --f32 --tune f32_pairs=3 --tune stream_ncw=15 > $O/ncu.log 2>&1
for r in $O/ncu_*.ncu-rep; do
  b=${r%.ncu-rep}
  ncu -i $r --page raw --csv > $b.raw.csv 2>/dev/null
  ncu -i $r --page details --csv > $b.details.csv 2>/dev/null
  ncu -i $r --page source --csv --print-source sass > $b.sass.csv 2>/dev/null
  gzip -f $b.sass.csv
  rm -f $r
done
ls -la $O
