# c4 / c4potts final lines + ncu of both packed kernels (instruction counts for the issue roofline)
mkdir -p gpurun_out/c4f
O=gpurun_out/c4f
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gibbs_packed -s 2 -c 1 -o $O/ncu_ising -f python tools/prof_ising.py > $O/ncu_i.log 2>&1; echo "ncu ising rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gibbs_packed -s 2 -c 1 -o $O/ncu_potts -f python tools/prof_ising.py --potts > $O/ncu_p.log 2>&1; echo "ncu potts rc=$?"
