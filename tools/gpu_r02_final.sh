# r02 final refresh: smoke, every GPU test, every bench line (default c1 with the reference
# cpu_baseline, all configs, reference arm, rank path), c1 launch list
O=gpurun_out/r02final
mkdir -p $O
: > $O/summary.txt
timeout 600 python __graft_entry__.py --smoke > $O/smoke.log 2>&1; echo "smoke rc=$? $(tail -1 $O/smoke.log)" >> $O/summary.txt
timeout 900 python bench.py > $O/bench_c1.log 2>&1; echo "c1 rc=$?" >> $O/summary.txt
for c in c0 c1f32 c2 c3 c3sweep c4 c4potts rng; do
  timeout 900 python bench.py --config $c > $O/bench_$c.log 2>&1; echo "$c rc=$?" >> $O/summary.txt
done
timeout 900 python bench.py --impl reference > $O/bench_reference_c1.log 2>&1; echo "reference rc=$?" >> $O/summary.txt
timeout 900 python bench.py --force-dist --exchange peer --no-cpu-baseline > $O/bench_c1_rankpath_peer.log 2>&1; echo "peer rc=$?" >> $O/summary.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c1.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1; echo "launch list rc=$?" >> $O/summary.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c1f32.csv python bench.py --config c1f32 --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch_f32.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c0.csv python bench.py --config c0 --steps 5 --warmup 3 --no-cpu-baseline > $O/ncu_launch_c0.log 2>&1
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > $O/pytest.log 2>&1; echo "pytest rc=$? $(tail -1 $O/pytest.log)" >> $O/summary.txt
cat $O/summary.txt
