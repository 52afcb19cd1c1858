# r02 pass S: packed Gibbs kernel, RPT consecutive rows per thread (tune gibbs_rpt): parity tests + A/B
O=gpurun_out/r02s
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_ising.py tests/test_gpu_denoise.py tests/test_gpu_multiproc.py -m gpu -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$? $(tail -1 $O/pytest.log)" > $O/summary.txt
for t in 4 2 1 4 1; do timeout 600 python bench.py --config c4 --no-cpu-baseline --tune gibbs_rpt=$t >> $O/c4_rpt$t.log 2>&1; done
for t in 4 2 1; do timeout 600 python bench.py --config c4potts --no-cpu-baseline --tune gibbs_rpt=$t >> $O/c4p_rpt$t.log 2>&1; done
cat $O/summary.txt
