# c4 / c4potts bench lines (with CPU baseline) + ncu full of one Ising and one Potts packed half-sweep
mkdir -p gpurun_out
timeout 900 python bench.py --config c4 > gpurun_out/bench_c4.log 2>&1; echo "c4 rc=$?"
timeout 900 python bench.py --config c4potts > gpurun_out/bench_c4potts.log 2>&1; echo "c4potts rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gibbs_packed -s 2 -c 1 -o gpurun_out/ncu_ising_final -f python tools/prof_ising.py > gpurun_out/ncu_if.log 2>&1; echo "ncu ising rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gibbs_packed -s 2 -c 1 -o gpurun_out/ncu_potts_final -f python tools/prof_ising.py --potts > gpurun_out/ncu_pf.log 2>&1; echo "ncu potts rc=$?"
