# r02 pass P: HB rows kernel with 8 self-producing consumer warps (default) vs 7 + idle warp
O=gpurun_out/r02p
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_hb.py tests/test_gpu_hb_sweep.py tests/test_gpu_protocols.py -m gpu -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$? $(tail -1 $O/pytest.log)" > $O/summary.txt
for t in 8 7 8 7; do timeout 600 python bench.py --config c3 --no-cpu-baseline --tune hb_rows_ncw=$t >> $O/c3_ncw$t.log 2>&1; done
for tps in 1 3 4; do timeout 600 python bench.py --config c3 --no-cpu-baseline --tune hb_rows_tps=$tps > $O/c3_ncw8_tps$tps.log 2>&1; done
cat $O/summary.txt
