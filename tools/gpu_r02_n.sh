# r02 pass N: F2F share A/B for the row-dot gradient phase + ncu source capture of the default fp32-X kernel
O=gpurun_out/r02n
mkdir -p $O
for v in 0 2; do
  PM_LIB_PATH=$PWD/paper_1310_1537_b200/libpmb200_F2F$v.so timeout 600 python bench.py --config c1f32 --no-cpu-baseline --steps 300 > $O/c1f32_f2f$v.log 2>&1
done
timeout 600 python bench.py --config c1f32 --no-cpu-baseline --steps 300 > $O/c1f32_f2f1.log 2>&1
timeout 300 python tools/prof_glm.py --f32 > $O/plain.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:glm_stream -s 3 -c 1 \
    -o $O/ncu_f32_rowdot16 -f python tools/prof_glm.py --f32 > $O/ncu.log 2>&1
for r in $O/ncu_*.ncu-rep; do
  b=${r%.ncu-rep}
  ncu -i $r --page raw --csv > $b.raw.csv 2>/dev/null
  ncu -i $r --page details --csv > $b.details.csv 2>/dev/null
  ncu -i $r --page source --csv --print-source sass > $b.sass.csv 2>/dev/null
  gzip -f $b.sass.csv
  rm -f $r
done
ls $O
