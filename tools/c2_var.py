"""Repeatability of the resident chain (config 2 shape): several identical 20-iteration runs."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1310_1537_b200 import glm  # noqa: E402
from paper_1310_1537_b200.sampler import ChainConfig, GaussianPrior, run_chain  # noqa: E402
from paper_1310_1537_b200.synthetic import baseline_design  # noqa: E402

x, y, _, _ = baseline_design(1_000_000, 50, seed=2)
d = glm.DesignMatrix(x, y)
p = GaussianPrior.isotropic(50, 0.0, 10.0)
for i in range(10):
    t0 = time.perf_counter()
    out = run_chain(d, p, ChainConfig(n_iter=20, n_burnin=0, seed=5))
    print(f"run {i} wall {out.wall_time:.4f} it/s {20 / out.wall_time:.1f} evals {out.accept_evals}", flush=True)
    if i == 4:
        time.sleep(2.0)
