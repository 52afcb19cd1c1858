"""Config-0 shape (N=1e5, K=32): the GLM stream kernel vs the HB row-per-lane kernel with
one group (offsets [0, N]); warm back-to-back launches and results compared."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1310_1537_b200 import glm as pglm  # noqa: E402
from paper_1310_1537_b200.hb import CsrGroups  # noqa: E402
from paper_1310_1537_b200.sampler import GaussianPrior  # noqa: E402
from paper_1310_1537_b200.synthetic import baseline_design  # noqa: E402

for n, k in [(100000, 32), (100000, 20), (1000000, 32), (10000, 32)]:
    x, y, _, betas = baseline_design(n, k, seed=1, n_eval=1)
    prior = GaussianPrior.isotropic(k, 0.0, 10.0)
    data = pglm.DesignMatrix(x, y)
    dev = data.on_device(0, "f64")
    dev.set_prior(prior.mu, prior.sigma)
    bl = np.random.default_rng(9).normal(0, 0.1, (200, k))
    dev.time_launches(bl[:20], with_prior=True, want_grad=True)
    t_glm = dev.time_launches(bl, with_prior=True, want_grad=True) / 200
    res = pglm.log_posterior_grad(data, bl[0], prior)
    hb = CsrGroups(x, y, np.array([0, n], dtype=np.int64)).on_device(0)
    f, g = hb.eval(bl[:1], prior.mu, prior.sigma)
    t_hb = 0.0
    hb.time_evals(bl[:1], prior.mu, prior.sigma, n=20)
    t_hb = hb.time_evals(bl[:1], prior.mu, prior.sigma, n=200) / 200
    print(f"N={n} K={k}: stream {t_glm*1e3:.2f} us, hb rows (G=1) {t_hb*1e3:.2f} us, "
          f"rel df {abs(f[0]-res.f)/abs(res.f):.2e}, max rel dg {np.max(np.abs(g[0]-res.g)/np.maximum(np.abs(res.g),1)):.2e}")
    hb.close()
