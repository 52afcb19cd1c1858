"""Small driver for ncu captures of the GLM stream kernel (config 1 shape by default).

python tools/prof_glm.py [--n N] [--k K] [--f32] [--launches L]
"""
import argparse
import os
import sys


sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1310_1537_b200 import glm  # noqa: E402
from paper_1310_1537_b200.sampler import GaussianPrior  # noqa: E402
from paper_1310_1537_b200.synthetic import baseline_design  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--n", type=int, default=10_000_000)
p.add_argument("--k", type=int, default=100)
p.add_argument("--f32", action="store_true")
p.add_argument("--launches", type=int, default=5)
p.add_argument("--tune", action="append", default=[])
a = p.parse_args()
from paper_1310_1537_b200 import _lib  # noqa: E402
for kv in a.tune:
    _lib.set_tune(kv.split("=")[0], int(kv.split("=")[1]))
x, y, _, betas = baseline_design(a.n, a.k, seed=1, n_eval=a.launches + 1)
d = glm.DesignMatrix(x, y)
prior = GaussianPrior.isotropic(a.k, 0.0, 10.0)
plan = glm.ExecPlan(x_storage="f32" if a.f32 else "f64")
for i in range(a.launches):
    r = glm.log_posterior_grad(d, betas[i], prior, plan)
print("f", r.f, "geometry", d.on_device(0, plan.x_storage).geometry())
