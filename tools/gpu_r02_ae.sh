# r02 pass AE: Gibbs compare on the FMA pipe (-DPM_AB_GIBBS_BORROW): bit-exact tests on the variant + c4 A/B
O=gpurun_out/r02ae
mkdir -p $O
PM_LIB_PATH=$PWD/paper_1310_1537_b200/libpmb200_BORROW.so timeout 900 python -m pytest tests/test_gpu_ising.py tests/test_gpu_denoise.py -m gpu -q -p no:cacheprovider > $O/pytest_borrow.log 2>&1; echo "pytest(borrow) rc=$? $(tail -1 $O/pytest_borrow.log)" > $O/summary.txt
for i in 1 2; do
  timeout 600 python bench.py --config c4 --no-cpu-baseline >> $O/c4_default.log 2>&1
  PM_LIB_PATH=$PWD/paper_1310_1537_b200/libpmb200_BORROW.so timeout 600 python bench.py --config c4 --no-cpu-baseline >> $O/c4_borrow.log 2>&1
done
cat $O/summary.txt
for f in c4_default c4_borrow; do grep '^{' $O/$f.log | python -c "
import sys,json
for line in sys.stdin:
    l=json.loads(line); print('$f', round(l['value'],1), 'sweeps/s', round(l['ms_per_step']*1e3,2), 'us')"; done
