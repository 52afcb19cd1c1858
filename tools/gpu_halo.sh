# peer-memory halo exchange: ising/dist GPU tests + c4 bench (exchange code path must not slow the plain kernel)
mkdir -p gpurun_out
: > gpurun_out/halo.txt
for t in test_gpu_ising test_gpu_dist test_gpu_denoise; do
  timeout 900 python -m pytest tests/$t.py -m gpu -q -x > gpurun_out/th_$t.log 2>&1; echo "$t rc=$? $(tail -1 gpurun_out/th_$t.log)" >> gpurun_out/halo.txt
done
for c in c4 c4potts; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/bh_$c.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/bh_$c.log').read().strip().splitlines()[-1]); print('$c', round(d['value'],1), d['unit'], round(d['ms_per_step']*1000,2), 'us/step')" >> gpurun_out/halo.txt 2>&1
done
cat gpurun_out/halo.txt
