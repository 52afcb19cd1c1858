# r02 profiling pass: c0 fixed-cost breakdown (A/B builds) + ncu source-level captures of
# the c0 stream kernel, the c1 fp32-X kernel and the packed Ising half-sweep
set -x
O=gpurun_out/p02
mkdir -p $O
for v in default EMPTY NO_FINALIZE NO_COMPUTE OUT_DEVICE; do
  if [ $v = default ]; then L=""; else L="PM_LIB_PATH=$PWD/paper_1310_1537_b200/libpmb200_$v.so"; fi
  env $L timeout 300 python tools/c0_breakdown.py --tag $v >> $O/c0_breakdown.jsonl 2>> $O/c0_breakdown.err
done
timeout 300 python tools/prof_glm.py --n 100000 --k 32 > $O/plain_c0.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:glm_stream -s 3 -c 1 \
    -o $O/ncu_c0 -f python tools/prof_glm.py --n 100000 --k 32 > $O/ncu_c0.log 2>&1
timeout 300 python tools/prof_glm.py --f32 > $O/plain_f32.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:glm_stream -s 3 -c 1 \
    -o $O/ncu_f32 -f python tools/prof_glm.py --f32 > $O/ncu_f32.log 2>&1
timeout 300 python tools/prof_ising.py > $O/plain_ising.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:gibbs_packed -s 2 -c 1 \
    -o $O/ncu_ising -f python tools/prof_ising.py > $O/ncu_ising.log 2>&1
# keep only the CSV pages (the .ncu-rep files exceed gpurun's 64 MiB return limit)
for r in $O/ncu_*.ncu-rep; do
  b=${r%.ncu-rep}
  ncu -i $r --page raw --csv > $b.raw.csv 2>/dev/null
  ncu -i $r --page details --csv > $b.details.csv 2>/dev/null
  ncu -i $r --page source --csv --print-source sass > $b.sass.csv 2>/dev/null
  gzip -f $b.sass.csv
  rm -f $r
done
du -sh $O
echo done
