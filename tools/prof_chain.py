"""Small driver for ncu captures of the device-resident chain kernel (config 2 shape)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1310_1537_b200 import glm  # noqa: E402
from paper_1310_1537_b200.sampler import ChainConfig, GaussianPrior, run_chain  # noqa: E402
from paper_1310_1537_b200.synthetic import baseline_design  # noqa: E402

n_iter = int(sys.argv[1]) if len(sys.argv) > 1 else 1
x, y, _, _ = baseline_design(1_000_000, 50, seed=2)
d = glm.DesignMatrix(x, y)
out = run_chain(d, GaussianPrior.isotropic(50, 0.0, 10.0), ChainConfig(n_iter=n_iter, n_burnin=0, seed=5))
print("evals", out.accept_evals, "passes", out.device_passes, "wall", out.wall_time)
