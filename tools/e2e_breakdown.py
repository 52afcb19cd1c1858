"""Config-0 end-to-end cost split: the public Python call vs the bare C-ABI call vs device time.

python tools/e2e_breakdown.py [--n 100000] [--k 32]
"""
import argparse
import ctypes
import json
import os
import statistics
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1310_1537_b200 import _lib, glm  # noqa: E402
from paper_1310_1537_b200.sampler import GaussianPrior  # noqa: E402
from paper_1310_1537_b200.synthetic import baseline_design  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--n", type=int, default=100_000)
p.add_argument("--k", type=int, default=32)
a = p.parse_args()
x, y, _, betas = baseline_design(a.n, a.k, seed=1, n_eval=256)
d = glm.DesignMatrix(x, y)
prior = GaussianPrior.isotropic(a.k, 0.0, 10.0)
dev = d.on_device(0)
dev.set_prior(prior.mu, prior.sigma)
lib = _lib.load()


def med(fn, n=2000):
    for i in range(50):
        fn(i)
    ts = []
    for i in range(n):
        t0 = time.perf_counter()
        fn(i)
        ts.append(time.perf_counter() - t0)
    return round(statistics.median(ts) * 1e6, 2)


f = ctypes.c_double()
g = np.empty(a.k)
gp = _lib.dptr(g)
bps = [_lib.dptr(np.ascontiguousarray(b)) for b in betas]
fp = ctypes.byref(f)
res = {
    "public_api_us": med(lambda i: glm.log_posterior_grad(d, betas[i & 255], prior)),
    "device_eval_method_us": med(lambda i: dev.eval(betas[i & 255], True, True)),
    "bare_c_call_us": med(lambda i: lib.pm_glm_eval(dev._h, bps[i & 255], 1, 1, fp, gp)),
    "device_warm_us": round(dev.time_launches(betas[:64], True, True) / 64 * 1e3, 2),
}
for t in (0,):
    _lib.set_tune("glm_poll", t)
    res[f"bare_c_call_sync_us"] = med(lambda i: lib.pm_glm_eval(dev._h, bps[i & 255], 1, 1, fp, gp))
    _lib.set_tune("glm_poll", None)
print(json.dumps(res))
