"""Per-call latency of the differential update vs the full evaluation at the reference's
acceptance-criterion-3 shape (N=200000, K=50; test_acceptance.py:92-125): wall-clock
medians of each public call, for the A/B of the diff path's fixed costs."""
import os
import statistics
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1310_1537_b200 import glm  # noqa: E402
from paper_1310_1537_b200.sampler import GaussianPrior, log_posterior_coord  # noqa: E402

data, _ = glm.synthetic_logistic(200_000, 50, seed=301)
prior = GaussianPrior.isotropic(50, sigma=5.0)
beta0 = np.random.default_rng(302).normal(0.0, 0.3, 50)
ws = glm.GlmWorkspace(data, beta0)
plan = glm.ExecPlan(glm.Strategy.PLF, workers=1)


def med(fn, n=200):
    for _ in range(10):
        fn()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts) * 1e6


b = beta0.copy()
print({"loglike_grad_us": med(lambda: glm.loglike_grad(data, b)),
       "loglike_us": med(lambda: glm.loglike(data, b)),
       "diff_loglike_us": med(lambda: glm.diff_loglike(ws, data, 7, 0.1)),
       "coord_full_us": med(lambda: log_posterior_coord(ws, data, prior, 7, 0.1, plan, False)),
       "coord_diff_us": med(lambda: log_posterior_coord(ws, data, prior, 7, 0.1, plan, True))})
