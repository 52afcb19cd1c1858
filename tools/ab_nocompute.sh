# pipeline-only timing (consumers release each stage without computing) vs the real kernel
mkdir -p gpurun_out
: > gpurun_out/ab_nocompute.txt
L=$PWD/paper_1310_1537_b200
for c in c1 c1f32; do
  for lib in libpmb200.so libpm_nc.so; do
    PM_LIB_PATH=$L/$lib timeout 600 python bench.py --config $c --steps 200 --no-cpu-baseline > gpurun_out/bc_${c}_$lib.log 2>&1
    python -c "import json; d=json.loads(open('gpurun_out/bc_${c}_$lib.log').read().strip().splitlines()[-1]); print('$c $lib', round(d['roofline']['kernel_ms']*1000,1), 'us kernel', round(d['roofline']['achieved'],0), 'GB/s', d['clocks']['sm_mhz'])" >> gpurun_out/ab_nocompute.txt 2>&1
  done
done
for k in 8 20 40; do
  for lib in libpmb200.so libpm_nc.so; do
    PM_LIB_PATH=$L/$lib PM_GLM_ROWS=0 timeout 300 python - >> gpurun_out/ab_nocompute.txt 2>&1 <<PY
import numpy as np, sys
sys.path.insert(0, '.')
from paper_1310_1537_b200 import glm
from paper_1310_1537_b200.synthetic import baseline_design
n=10_000_000
for xs in ('f64','f32'):
    x, y, _, b = baseline_design(n, $k, seed=1, n_eval=20)
    d = glm.DesignMatrix(x, y)
    dev = d.on_device(0, xs)
    dev.time_launches(b[:3], False, True)
    ms = dev.time_launches(b, False, True) / len(b)
    bytes_ = n * ($k * (8 if xs == 'f64' else 4) + 8)
    print('K=$k', xs, '$lib', round(ms*1000,1), 'us', round(bytes_/ms/1e6), 'GB/s', dev.geometry())
    d.release_device()
PY
  done
done
cat gpurun_out/ab_nocompute.txt
