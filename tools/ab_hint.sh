# A/B of the mbarrier try_wait suspend-time hint and the small-K kernel choice on c0 / c1 / c3
mkdir -p gpurun_out
for v in "" _h0 _h2000 _h50000; do
  for rows in 1 0; do
    lib=paper_1310_1537_b200/libpmb200$v.so
    PM_LIB_PATH=$PWD/$lib PM_GLM_ROWS=$rows timeout 300 python bench.py --config c0 --steps 500 --no-cpu-baseline \
      > gpurun_out/ab_c0$v.rows$rows.log 2>&1
  done
  PM_LIB_PATH=$PWD/paper_1310_1537_b200/libpmb200$v.so timeout 300 python bench.py --config c1 --steps 200 --no-cpu-baseline > gpurun_out/ab_c1$v.log 2>&1
  PM_LIB_PATH=$PWD/paper_1310_1537_b200/libpmb200$v.so timeout 300 python bench.py --config c3 --steps 300 --no-cpu-baseline > gpurun_out/ab_c3$v.log 2>&1
done
for f in gpurun_out/ab_c*.log; do
  python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value'],1), round(d['ms_per_step']*1000,2), 'us')"
done > gpurun_out/ab_hint.txt
