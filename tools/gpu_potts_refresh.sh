# c4potts bench line (with CPU baseline) + ncu full of the Potts packed kernel (committed build)
mkdir -p gpurun_out
timeout 900 python bench.py --config c4potts > gpurun_out/bench_c4potts.log 2>&1; echo "c4potts rc=$?"
tail -1 gpurun_out/bench_c4potts.log | cut -c1-300
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gibbs_packed -s 2 -c 1 -o gpurun_out/ncu_potts_final -f python tools/prof_ising.py --potts > gpurun_out/ncu_pf.log 2>&1; echo "ncu rc=$?"
