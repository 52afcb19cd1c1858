# validation after the Gibbs changes: smoke, all GPU tests, c4/c4potts bench lines, ncu of the Potts kernel
mkdir -p gpurun_out
: > gpurun_out/val2.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/val2.txt
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/t_all_gpu.log 2>&1; echo "pytest -m gpu rc=$? $(tail -1 gpurun_out/t_all_gpu.log)" >> gpurun_out/val2.txt
timeout 900 python bench.py --config c4potts > gpurun_out/bench_c4potts.log 2>&1; echo "c4potts rc=$?" >> gpurun_out/val2.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gibbs_packed -s 2 -c 1 -o gpurun_out/ncu_potts_final -f python tools/prof_ising.py --potts > gpurun_out/ncu_pf.log 2>&1; echo "ncu potts rc=$?" >> gpurun_out/val2.txt
cat gpurun_out/val2.txt
