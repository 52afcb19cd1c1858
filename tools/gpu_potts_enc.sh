mkdir -p gpurun_out/pe
O=gpurun_out/pe
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gibbs_packed -s 2 -c 1 -o $O/ncu_potts -f python tools/prof_ising.py --potts > $O/ncu_p.log 2>&1; echo "ncu potts rc=$?"
