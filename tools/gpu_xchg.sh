# peer-memory exchange: GPU tests + rank-path bench at N=1 (peer vs NCCL) + plain c1
mkdir -p gpurun_out
: > gpurun_out/xchg.txt
timeout 600 python -m pytest tests/test_gpu_dist.py -m gpu -q -x > gpurun_out/t_dist.log 2>&1; echo "dist tests rc=$?" >> gpurun_out/xchg.txt
tail -2 gpurun_out/t_dist.log >> gpurun_out/xchg.txt
timeout 900 python -m pytest tests/test_gpu_glm.py -m gpu -q -x > gpurun_out/t_glm.log 2>&1; echo "glm tests rc=$?" >> gpurun_out/xchg.txt
for v in "peer --force-dist --exchange peer" "nccl --force-dist --exchange nccl" "plain"; do
  set -- $v; name=$1; shift
  timeout 600 python bench.py --steps 300 --no-cpu-baseline "$@" > gpurun_out/bx_$name.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/bx_$name.log').read().strip().splitlines()[-1]); print('$name', round(d['value'],1), round(d['ms_per_step']*1000,1), 'us/step kernel', round(d['roofline']['kernel_ms']*1000,1), 'e2e', round(d['e2e']['value'],1), d['gpu_launches'], d['config'].get('collective','-')[:40])" >> gpurun_out/xchg.txt 2>&1
done
cat gpurun_out/xchg.txt
