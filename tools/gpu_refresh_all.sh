# round-end refresh: new Potts/Ising tests, every bench line (default c1 + all configs + reference arm + rank path), c1 launch list
mkdir -p gpurun_out/refresh
O=gpurun_out/refresh
: > $O/summary.txt
timeout 900 python -m pytest tests/test_gpu_ising.py -m gpu -q > $O/t_ising.log 2>&1; echo "test_gpu_ising rc=$? $(tail -1 $O/t_ising.log)" >> $O/summary.txt
timeout 900 python bench.py > $O/bench_c1.log 2>&1; echo "c1 rc=$?" >> $O/summary.txt
for c in c0 c1f32 c2 c3 c3sweep c4 c4potts rng; do
  timeout 900 python bench.py --config $c > $O/bench_$c.log 2>&1; echo "$c rc=$?" >> $O/summary.txt
done
timeout 900 python bench.py --impl reference > $O/bench_reference_c1.log 2>&1; echo "reference rc=$?" >> $O/summary.txt
timeout 900 python bench.py --force-dist --exchange peer --no-cpu-baseline > $O/bench_c1_rankpath_peer.log 2>&1; echo "peer rc=$?" >> $O/summary.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c1.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1; echo "launch list rc=$?" >> $O/summary.txt
cat $O/summary.txt
