"""A/B: row-per-lane vs column-per-lane flat GLM kernel over small even K (N = 1e7 and 1e5)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1310_1537_b200 import glm  # noqa: E402

for n in (10_000_000, 100_000):
    for k in (4, 8, 16, 20, 24, 30, 32):
        gen = np.random.default_rng(k)
        x = gen.standard_normal((n, k))
        y = (gen.random(n) < 0.5).astype(float)
        betas = gen.normal(0, 0.1, (50, k))
        res = {}
        for rows in ("1", "0"):
            os.environ["PM_GLM_ROWS"] = rows
            d = glm.DesignMatrix(x, y)
            dev = d.on_device(0)
            dev.time_launches(betas[:5], False, True)
            ms = dev.time_launches(betas, False, True) / len(betas)
            res[dev.geometry()["kernel"]] = ms
            d.release_device()
        gbs = {kk: n * (k * 8 + 8) / (v * 1e-3) / 1e9 for kk, v in res.items()}
        print(n, k, {kk: round(v * 1e3, 1) for kk, v in res.items()}, "us", {kk: round(v) for kk, v in gbs.items()},
              "GB/s", flush=True)
