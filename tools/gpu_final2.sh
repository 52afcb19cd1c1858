mkdir -p gpurun_out/f2
O=gpurun_out/f2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1200 python -m pytest tests -m gpu -q > $O/t_gpu.log 2>&1; echo "pytest -m gpu rc=$? $(tail -1 $O/t_gpu.log)"
for c in c4 c4potts; do timeout 900 python bench.py --config $c > $O/bench_$c.log 2>&1; echo "$c rc=$?"; done
