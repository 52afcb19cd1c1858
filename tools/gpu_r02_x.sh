# r02 pass X: self-producing column consumers (8 warps) in the stream kernel: parity + c0 A/B
O=gpurun_out/r02x
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_glm.py tests/test_gpu_protocols.py tests/test_gpu_hb.py tests/test_gpu_dist.py -m gpu -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$? $(tail -1 $O/pytest.log)" > $O/summary.txt
for sp in 1 0; do for tps in 0 1 2 3; do
  T="--tune stream_selfprod=$sp"; if [ $tps != 0 ]; then T="$T --tune stream_tps=$tps"; fi
  timeout 300 python tools/c0_breakdown.py --tag sp${sp}_tps$tps $T >> $O/c0_breakdown.jsonl 2>> $O/c0.err
done; done
for sp in 1 0 1 0; do timeout 600 python bench.py --config c0 --no-cpu-baseline --tune stream_selfprod=$sp >> $O/c0_sp$sp.log 2>&1; done
cat $O/summary.txt
