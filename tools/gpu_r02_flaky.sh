# flakiness check: the protocol / multi-process / thread tests five times over
O=gpurun_out/r02flaky
mkdir -p $O
: > $O/summary.txt
for i in 1 2 3 4 5; do
  timeout 900 python -m pytest tests/test_gpu_multiproc.py tests/test_gpu_protocols.py tests/test_abi.py tests/test_gpu_dist.py -m gpu -q -p no:cacheprovider > $O/pytest_$i.log 2>&1; echo "run $i rc=$? $(tail -1 $O/pytest_$i.log)" >> $O/summary.txt
done
cat $O/summary.txt
