# r02 pass A: smoke, full GPU test suite, default bench (c1) + reference arm, launch list and
# one ncu --set full capture of the c1 stream kernel (raw/details CSV pages only)
O=gpurun_out/r02a
mkdir -p $O
: > $O/summary.txt
timeout 600 python __graft_entry__.py --smoke > $O/smoke.log 2>&1; echo "smoke rc=$? $(tail -1 $O/smoke.log)" >> $O/summary.txt
timeout 900 python bench.py > $O/bench_c1.log 2>&1; echo "c1 rc=$?" >> $O/summary.txt
timeout 900 python bench.py --impl reference > $O/bench_reference_c1.log 2>&1; echo "reference rc=$?" >> $O/summary.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c1.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1; echo "launch list rc=$?" >> $O/summary.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:glm_stream -s 3 -c 1 -o $O/ncu_c1 -f python tools/prof_glm.py > $O/ncu_c1.log 2>&1; echo "ncu c1 rc=$?" >> $O/summary.txt
for r in $O/ncu_*.ncu-rep; do
  b=${r%.ncu-rep}
  ncu -i $r --page raw --csv > $b.raw.csv 2>/dev/null
  ncu -i $r --page details --csv > $b.details.csv 2>/dev/null
  rm -f $r
done
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=25 > $O/pytest.log 2>&1; echo "pytest rc=$? $(tail -1 $O/pytest.log)" >> $O/summary.txt
cat $O/summary.txt
