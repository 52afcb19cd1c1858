"""Config-0 fixed-cost breakdown: warm back-to-back launches (pm_glm_time_launches) and
single cold launches (L2 scrubbed) at several N, for the library named by PM_LIB_PATH
(A/B builds: -DPM_AB_EMPTY, -DPM_AB_NO_FINALIZE, -DPM_AB_NO_COMPUTE, -DPM_AB_OUT_DEVICE).

python tools/c0_breakdown.py [--tag NAME] [--k 32] [--tune knob=v ...]
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1310_1537_b200 import _lib, glm  # noqa: E402
from paper_1310_1537_b200.sampler import GaussianPrior  # noqa: E402
from paper_1310_1537_b200.synthetic import baseline_design  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--tag", default=os.path.basename(os.environ.get("PM_LIB_PATH", "default")))
p.add_argument("--k", type=int, default=32)
p.add_argument("--tune", action="append", default=[])
a = p.parse_args()
for kv in a.tune:
    knob, v = kv.split("=")
    _lib.set_tune(knob, int(v))
import torch  # noqa: E402

scrub = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
clean = torch.ones(256 << 20, dtype=torch.uint8, device="cuda")
res = {"tag": a.tag, "k": a.k, "tune": a.tune}
for n in (32, 4096, 100_000, 1_000_000):
    x, y, _, betas = baseline_design(n, a.k, seed=1, n_eval=64)
    d = glm.DesignMatrix(x, y)
    dev = d.on_device(0)
    prior = GaussianPrior.isotropic(a.k, 0.0, 10.0)
    dev.set_prior(prior.mu, prior.sigma)
    dev.time_launches(betas[:8], True, True)
    warm = [dev.time_launches(betas, True, True) / len(betas) for _ in range(3)]
    cold = []
    for i in range(20):
        scrub.zero_()
        clean.max()
        torch.cuda.synchronize()
        cold.append(dev.time_launches(betas[i:i + 1], True, True))
    cold_dev = dev.time_cold(betas[:20], True, True) / 20  # scrub on the launching stream
    res[str(n)] = {"warm_us": round(min(warm) * 1e3, 2), "cold_us_median": round(float(np.median(cold)) * 1e3, 2),
                   "cold_dev_us": round(cold_dev * 1e3, 2), "geometry": dev.geometry()}
    d.release_device()
print(json.dumps(res))
