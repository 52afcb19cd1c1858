O=gpurun_out/r02v
mkdir -p $O
timeout 300 python tools/e2e_breakdown.py > $O/e2e_c0.json 2> $O/e2e.err
timeout 300 python tools/e2e_breakdown.py --n 32 --k 32 > $O/e2e_n32.json 2>> $O/e2e.err
cat $O/e2e_c0.json $O/e2e_n32.json; tail -3 $O/e2e.err
