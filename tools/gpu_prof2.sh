mkdir -p gpurun_out
timeout 300 python tools/prof_ising.py > gpurun_out/p1.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gibbs_packed -s 1 -c 1 -o gpurun_out/ncu_gibbs2 -f python tools/prof_ising.py > gpurun_out/n1.log 2>&1; echo "ising rc=$?"
timeout 300 python tools/prof_chain.py 1 > gpurun_out/p2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --replay-mode application -k regex:chain -c 1 -o gpurun_out/ncu_chain -f python tools/prof_chain.py 1 > gpurun_out/n2.log 2>&1; echo "chain rc=$?"
tail -5 gpurun_out/n2.log
