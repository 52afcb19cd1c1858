mkdir -p gpurun_out
for rep in 1 2 3; do for u in 1 2; do
  echo "rep=$rep U=$u $(PM_CHAIN_UNROLL=$u timeout 300 python tools/prof_chain.py 20 2>&1 | tail -1)" >> gpurun_out/ab_chain2.txt
done; done
python - <<'PY' >> gpurun_out/ab_chain2.txt 2>&1
import os, sys, time
sys.path.insert(0, '.')
from paper_1310_1537_b200 import glm
from paper_1310_1537_b200.sampler import ChainConfig, GaussianPrior, run_chain
from paper_1310_1537_b200.synthetic import baseline_design
x, y, _, _ = baseline_design(1_000_000, 50, seed=2)
d = glm.DesignMatrix(x, y)
p = GaussianPrior.isotropic(50, 0.0, 10.0)
for i in range(6):
    out = run_chain(d, p, ChainConfig(n_iter=20, n_burnin=0, seed=5 + i))
    print('in-process run', i, 'evals', out.accept_evals, 'wall', round(out.wall_time, 4), 'it/s', round(20 / out.wall_time, 1))
PY
cat gpurun_out/ab_chain2.txt
