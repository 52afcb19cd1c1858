# r02 pass B: every other bench line, c0 fixed-cost breakdown over the A/B builds, the Gibbs
# shared-memory staging A/B, ncu source-level captures (c0, c1 fp32-X, packed Ising, HB rows),
# compute-sanitizer (memcheck, racecheck, synccheck) over tools/sanitize_subset.py
O=gpurun_out/r02b
mkdir -p $O
: > $O/summary.txt
for c in c0 c1f32 c2 c3 c3sweep c4 c4potts rng; do
  timeout 900 python bench.py --config $c > $O/bench_$c.log 2>&1; echo "$c rc=$?" >> $O/summary.txt
done
timeout 900 python bench.py --force-dist --exchange peer --no-cpu-baseline > $O/bench_c1_rankpath_peer.log 2>&1; echo "peer rc=$?" >> $O/summary.txt
for v in default EMPTY NO_FINALIZE NO_COMPUTE PHASES; do
  if [ $v = default ]; then L=""; else L="PM_LIB_PATH=$PWD/paper_1310_1537_b200/libpmb200_$v.so"; fi
  env $L timeout 300 python tools/c0_breakdown.py --tag $v >> $O/c0_breakdown.jsonl 2>> $O/c0_breakdown.err
done
for t in 0 1; do timeout 600 python bench.py --config c4 --steps 1000 --warmup 10 --no-cpu-baseline --tune gibbs_smem=$t > $O/c4_smem$t.log 2>&1; done
for t in 0 1; do timeout 600 python bench.py --config c4potts --steps 1000 --warmup 10 --no-cpu-baseline --tune gibbs_smem=$t > $O/c4p_smem$t.log 2>&1; done
timeout 300 python tools/prof_glm.py --n 100000 --k 32 > $O/plain_c0.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:glm_stream -s 3 -c 1 \
    -o $O/ncu_c0 -f python tools/prof_glm.py --n 100000 --k 32 > $O/ncu_c0.log 2>&1
timeout 300 python tools/prof_glm.py --f32 > $O/plain_f32.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:glm_stream -s 3 -c 1 \
    -o $O/ncu_f32 -f python tools/prof_glm.py --f32 > $O/ncu_f32.log 2>&1
timeout 300 python tools/prof_ising.py > $O/plain_ising.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:gibbs_packed -s 2 -c 1 \
    -o $O/ncu_ising -f python tools/prof_ising.py > $O/ncu_ising.log 2>&1
timeout 300 python tools/prof_hb.py > $O/plain_hb.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:hb_rows -s 2 -c 1 \
    -o $O/ncu_hb -f python tools/prof_hb.py > $O/ncu_hb.log 2>&1
for r in $O/ncu_*.ncu-rep; do
  b=${r%.ncu-rep}
  ncu -i $r --page raw --csv > $b.raw.csv 2>/dev/null
  ncu -i $r --page details --csv > $b.details.csv 2>/dev/null
  ncu -i $r --page source --csv --print-source sass > $b.sass.csv 2>/dev/null
  gzip -f $b.sass.csv
  rm -f $r
done
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_subset.py > $O/sanitizer_$tool.log 2>&1
  echo "sanitizer $tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $O/sanitizer_$tool.log | tail -1)" >> $O/summary.txt
done
du -sh $O
cat $O/summary.txt
