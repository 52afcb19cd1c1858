# r02 pass O: HB rows kernel with self-producing consumer warps (tune hb_selfprod) + HB tests
O=gpurun_out/r02o
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_hb.py tests/test_gpu_hb_sweep.py -m gpu -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$? $(tail -1 $O/pytest.log)" > $O/summary.txt
for t in 1 0 1 0; do timeout 600 python bench.py --config c3 --no-cpu-baseline --tune hb_selfprod=$t >> $O/c3_selfprod$t.log 2>&1; done
for tps in 1 2 4; do timeout 600 python bench.py --config c3 --no-cpu-baseline --tune hb_selfprod=1 --tune hb_rows_tps=$tps > $O/c3_self_tps$tps.log 2>&1; done
cat $O/summary.txt
