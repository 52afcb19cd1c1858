mkdir -p gpurun_out/c4e
O=gpurun_out/c4e
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gibbs_packed -s 2 -c 1 -o $O/ncu_ising -f python tools/prof_ising.py > $O/ncu_i.log 2>&1; echo "ncu ising rc=$?"
