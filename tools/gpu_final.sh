# round validation: every GPU test file, smoke, default bench (+cpu baseline), reference arm,
# rank path with the in-kernel peer exchange, c4 with the issue roofline, launch list + ncu of c1
mkdir -p gpurun_out
: > gpurun_out/final.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/final.txt
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/t_all_gpu.log 2>&1; echo "pytest -m gpu rc=$? $(tail -1 gpurun_out/t_all_gpu.log)" >> gpurun_out/final.txt
timeout 900 python bench.py > gpurun_out/bench_c1.log 2>&1; echo "bench rc=$?" >> gpurun_out/final.txt
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo "bench ref rc=$?" >> gpurun_out/final.txt
timeout 900 python bench.py --force-dist --exchange peer --no-cpu-baseline > gpurun_out/bench_c1_peer.log 2>&1; echo "bench peer rc=$?" >> gpurun_out/final.txt
timeout 900 python bench.py --config c4 > gpurun_out/bench_c4.log 2>&1; echo "bench c4 rc=$?" >> gpurun_out/final.txt
for f in bench_c1 bench_ref bench_c1_peer bench_c4; do tail -1 gpurun_out/$f.log | cut -c1-400 >> gpurun_out/final.txt; done
cat gpurun_out/final.txt
